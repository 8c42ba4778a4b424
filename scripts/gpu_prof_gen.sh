# full ncu capture (source-level) of the quantile-mode fused kernel at a reduced C3 sweep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/r02_genq${TAG:-} python bench.py --reps 2000 --steps 1 --warmup 0 --no-cpu-baseline --no-trace --no-ab --no-c5 > gpurun_out/r02_ncu_genq${TAG:-}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r02_ncu_genq${TAG:-}.log; ls -la gpurun_out/
