"""bench.py -- simulated requests/s on the MBB k x B x lambda sweep (BASELINE.json).

Workload ("C3", BASELINE.json configs[2]): k in {1,2,4,8,16} x B in {8,16,32}
x lambda in {0.5,0.6,0.7,0.8,0.9,0.95,0.99} of each point's capacity
throughput(B, k, a+b, a+1024b) (analytics.hpp:65-69), linear service
t = 0.03*len + 0.5 with len ~ U(1,1024) (tokens_to_time, workload.hpp:167-170),
uniform (equal-mass) bins, single server, flush on.  105 points x R
replications x 10^5 requests; one step = the whole sweep (all points, all
replications, per-point mean/std), fused generated-mode kernel (Philox).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1: launched by torch.distributed.run, one rank per GPU over NCCL.  Weak
scaling: every rank simulates R replications of every point
(replications [rank*R, (rank+1)*R) of an N*R-replication sweep, seeds
replication_seed(seed, r)) into its own block; the blocks are combined with
ONE NCCL all-gather and reduced per point in replication order exactly as
run_point does.

--impl reference: the unmodified reference engine (oracle/_ref/libbbref.so,
compiled from /root/reference's headers) on all host cores over a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

A_INTERCEPT, B_SLOPE = 0.5, 0.03
KS = [1, 2, 4, 8, 16]
BS = [8, 16, 32]
FRACS = [0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99]
SEED = 0x0000000241204504
METRIC = "simulated requests/s (MBB k×B×λ sweep) at 1/2/4/8 B200 vs CPU ref"
ALG_INSTR_BASE = 132.0  # lane-instructions per request, base case
ALG_INSTR_PER_BATCH = 12.0
# exact per-replication p50/p99 (the reference sorts every replication's
# latencies, simulator.hpp:289-301): the fused kernel logs (arrival fp64,
# batch id u32) per request and reads the log back once -- 24 B/request of
# HBM traffic that no log-based exact selection avoids
ALG_BYTES_QUANTILES = 24.0


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": True}  # B200_PROFILING.md fallback


def capacity(B, k, lo, hi):
    # analytics.hpp:55-69, expected_service_time / throughput
    mid = (lo + hi) / 2.0
    gap = (B * hi + lo) / (B + 1.0) - mid
    return B / (mid + gap / k)


def sweep_points(n_requests):
    lo_t = B_SLOPE * 1.0 + A_INTERCEPT
    hi_t = B_SLOPE * 1024.0 + A_INTERCEPT
    pts = []
    for k in KS:
        for B in BS:
            cap = capacity(B, k, lo_t, hi_t)
            for f in FRACS:
                pts.append(dict(k=k, B=B, lam=f * cap, n=n_requests))
    return pts


def alg_instr(points, reps):
    return sum((ALG_INSTR_BASE + ALG_INSTR_PER_BATCH / p["B"]) * p["n"] * reps for p in points)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons during the timed region (NVML, 100 ms)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# ------------------------------------------------------------- CPU reference
def reference_sample(points, reps, threads):
    """The unmodified reference engine (oracle/_ref) over `reps` replications
    of every point, on `threads` host threads.  Returns (requests, seconds)."""
    import concurrent.futures as cf

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O

    lib = O.reference()
    lo_t, hi_t = B_SLOPE + A_INTERCEPT, B_SLOPE * 1024 + A_INTERCEPT
    edges = {}
    for p in points:
        if p["k"] not in edges:
            edges[p["k"]] = O.uniform_boundaries(p["k"], lo_t, hi_t)
    jobs = [(p, r) for p in points for r in range(reps)]

    def one(job):
        p, r = job
        cfg = dict(arrival_rate=p["lam"], n_requests=p["n"], batch_size=p["B"],
                   edges=edges[p["k"]], service="linear", lo=1.0, hi=1024.0,
                   lin_a=A_INTERCEPT, lin_b=B_SLOPE)
        O.run_replicas(cfg, SEED, r, 1, 1)
        return p["n"]

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        total = sum(ex.map(one, jobs))
    return total, time.perf_counter() - t0
    del lib


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    pts = sweep_points(args.requests)
    reps = args.ref_reps
    for _ in range(args.warmup):
        reference_sample(pts[:: max(1, len(pts) // 15)], 1, threads)
    tot_req, tot_s = 0, 0.0
    for _ in range(args.steps):
        r, s = reference_sample(pts, reps, threads)
        tot_req += r
        tot_s += s
    v = tot_req / tot_s
    sample = (f"{len(pts)} C3 points x {reps} replication(s) x {args.requests} requests per step "
              f"(the full sweep uses {args.reps} replications per GPU)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "requests/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference mt19937_64 streams)",
        "config": workload_config(args, reps),
        "cpu_baseline": {"value": v, "unit": "requests/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "requests/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, reps):
    return {
        "workload": "C3 sweep (BASELINE configs[2]): k{1,2,4,8,16} x B{8,16,32} x "
                    "lambda{0.5,0.6,0.7,0.8,0.9,0.95,0.99} of capacity; linear service "
                    "t=0.03*len+0.5, len~U(1,1024); uniform equal-mass bins; 1 server; flush",
        "points": len(KS) * len(BS) * len(FRACS), "replications_per_gpu": reps,
        "requests_per_replication": args.requests,
        "requests_per_step_per_gpu": len(KS) * len(BS) * len(FRACS) * reps * args.requests,
        "rng": "Philox4x32-10 (counter-based), fp64 arrival clock and Lindley recursion",
        "quantiles": ("off (A/B run)" if getattr(args, "no_quantiles", False) else
                      "exact latency p50/p99 of every replication, averaged per point, as "
                      "run_point does (experiment.hpp:256-279)"),
        "l2": "no HBM-resident inputs in generated mode; a 512 MiB buffer is written between "
              "timed steps anyway (L2 flushed)",
        "parallelism": f"replicas sharded over {args.gpus} GPU(s), 1 NCCL all-gather per step",
    }


# ------------------------------------------------------------------- ours
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--reps", type=int, default=10_000, help="replications per point per GPU")
    ap.add_argument("--requests", type=int, default=100_000)
    ap.add_argument("--ref-reps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--no-quantiles", action="store_true",
                    help="A/B only: skip the per-replication p50/p99 the reference computes")
    ap.add_argument("--no-ab", action="store_true", help="skip the without-quantiles A/B leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 large-run sample")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 noisy-predictor grid")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default) or gloo for testing")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2412_04504_b200 as bb

    if args.no_quantiles:
        bb.set_generated_quantiles(False)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # functional testing of the N>1 path on a single GPU
            dist.init_process_group(args.dist_backend)
    # one explicit stream for torch's own ops and the engine's launches (the
    # engine's stream-ordered entries run on the stream they are handed; the
    # legacy default stream's handle is 0, which the C ABI reads as "the
    # library's own stream")
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream

    pts = sweep_points(args.requests)
    tpl = [bb.RunTemplate(arrival_rate=p["lam"], n_requests=p["n"], batch_size=p["B"],
                          bins=bb.BinRule(k=p["k"]),
                          service=bb.ServiceSpec("linear", 1.0, 1024.0, intercept=A_INTERCEPT,
                                                 slope=B_SLOPE)) for p in pts]
    P, R = len(tpl), args.reps
    Rtot = R * world
    block = torch.empty(6 * P * R, dtype=torch.float64, device=dev)  # this rank's replications
    gathered = torch.empty(6 * P * Rtot, dtype=torch.float64, device=dev) if world > 1 else block
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    results = {}

    from paper_2412_04504_b200 import dist as bbdist

    lo, hi = bbdist.weak_shard(R, rank)

    def step():
        bb.points_shard_local_device(tpl, Rtot, SEED, lo, hi, block.data_ptr(), sptr)
        bbdist.gather(block, gathered)  # the sweep's one NCCL all-gather (no-op at N=1)
        results["pts"] = bb.points_reduce_gathered_device(tpl, Rtot, world, gathered.data_ptr(), sptr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    bb.launch_count(reset=True)
    times, kern = [], []
    clocks = ClockSampler(local)
    with clocks:
        for _ in range(args.steps):
            flush.fill_(1)  # untimed L2 flush between timed steps
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            times.append(e0.elapsed_time(e1))
            kern.append(bb.last_kernel_ms()[0])
    launches = bb.launch_count()
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    requests_step = P * Rtot * args.requests
    value = requests_step * args.steps / (total_ms / 1e3)

    # e2e through the host-facing C ABI (spec from host, results on host)
    bb.transfer_bytes(reset=True)
    e2e_times = []
    for _ in range(max(1, min(args.steps, 3))):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            out = bb.run_points(tpl, R, SEED)
        else:
            step()
            out = results["pts"]
        e2e_times.append(time.perf_counter() - t0)
    h2d, d2h = bb.transfer_bytes()
    n_e2e = len(e2e_times)
    e2e_s = sum(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": requests_step * n_e2e / e2e_s, "unit": "requests/s",
           "h2d_bytes_per_step": int(h2d // n_e2e), "d2h_bytes_per_step": int(d2h // n_e2e),
           "api": "bb_run_points (host templates -> host PointResults)" if world == 1
           else "host spec -> shard -> NCCL all-gather -> reduce -> host PointResults"}
    # consistency: the e2e results equal the device-timed results
    same = all(a.throughput_mean == b.throughput_mean for a, b in zip(out, results["pts"]))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    ck = clocks.summary()
    kms = sorted(k for k in kern if k and k > 0)
    kernel_ms = kms[len(kms) // 2] if kms else None
    instr = alg_instr(pts, R)
    sm_mhz = ck.get("sm_mhz") or 1327.0
    peak = 148 * 4 * 32 * sm_mhz * 1e6
    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 6650.0) * 1e9
    quant = not args.no_quantiles
    roofline = None
    if kernel_ms:
        # two floors on one kernel: the simulation's instruction issue and,
        # with the quantiles, the request log's HBM traffic
        t_k = kernel_ms / 1e3
        t_issue = instr / peak
        qbytes = ALG_BYTES_QUANTILES * requests_step if quant else 0.0
        t_hbm = qbytes / hbm_peak
        traffic = None
        prof = latest_profile("gen_kernel_q_ncu.json" if quant else "gen_kernel_ncu.json")
        if prof:  # one `ncu --set full` capture; scaled per launch
            cap = json.load(open(prof))
            cap = cap[0] if isinstance(cap, list) else cap
            if cap.get("dram_bytes_per_request") is not None:
                traffic = cap["dram_bytes_per_request"] * requests_step
            elif cap.get("dram_bytes_per_launch") is not None:
                traffic = cap["dram_bytes_per_launch"] * R / 1500.0
        hbm_dom = t_hbm > t_issue
        roofline = {
            "bound": "hbm" if hbm_dom else "issue", "kernel": "gen_kernel",
            "achieved": (qbytes / t_k / 1e9) if hbm_dom else instr / t_k / 1e9,
            "peak": hbm_peak / 1e9 if hbm_dom else peak / 1e9,
            "unit": "GB/s" if hbm_dom else "Glane-instr/s",
            "frac": max(t_issue, t_hbm) / t_k, "traffic": traffic,
            "issue": {"achieved": instr / t_k / 1e9, "peak": peak / 1e9, "unit": "Glane-instr/s",
                      "frac": t_issue / t_k},
            "hbm": {"achieved": qbytes / t_k / 1e9, "peak": hbm_peak / 1e9, "unit": "GB/s",
                    "frac": t_hbm / t_k},
            "kernel_ms": kernel_ms, "kernel_share_of_step": kernel_ms / (total_ms / args.steps),
            "algorithmic": f"issue: {ALG_INSTR_BASE:.0f} + {ALG_INSTR_PER_BATCH:.0f}/B lane-instructions "
                           "per request (SURVEY 8d base case); hbm: "
                           + (f"{ALG_BYTES_QUANTILES:.0f} B/request (exact p50/p99: write + read the "
                              "12 B request log)" if quant else "none (quantiles off)")
                           + "; frac = max(issue time, HBM time) at peak / kernel time",
            "peak_basis": f"issue: 148 SM x 4 schedulers x 32 lanes x {sm_mhz} MHz (median SM "
                          "clock during the timed region); hbm: MEASURED_PEAKS.json",
        }
    line = {
        "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Philox4x32-10 streams generated on device)",
        "config": workload_config(args, R), "roofline": roofline,
        "e2e": e2e, "gpu_launches": int(launches), "clocks": ck,
        "results_consistent_e2e_vs_device": bool(same),
        "sample_point": {"k": results["pts"][-1].k, "B": results["pts"][-1].batch_size,
                         "throughput_mean": results["pts"][-1].throughput_mean,
                         "latency_mean": results["pts"][-1].latency_mean},
    }
    if world == 1 and quant and not args.no_ab:
        # A/B only: the same sweep without the per-replication quantiles
        bb.set_generated_quantiles(False)
        try:
            step()
            torch.cuda.synchronize()
            ab = []
            for _ in range(2):
                flush.fill_(1)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                torch.cuda.synchronize()
                ab.append(e0.elapsed_time(e1))
            line["without_quantiles"] = {
                "value": requests_step * len(ab) / (sum(ab) / 1e3), "unit": "requests/s",
                "note": "A/B only: p50/p99 left NaN, i.e. less work than the reference's run_point"}
        finally:
            bb.set_generated_quantiles(True)
    if world == 1 and not args.no_c4:
        try:
            line["c4_grid"] = c4_measure(bb, torch, stream)
        except Exception as e:  # secondary measurement; never fail the headline
            line["c4_grid"] = {"error": repr(e)}
    if world == 1 and not args.no_c5:
        try:
            line["c5_sample"] = c5_measure(bb, torch, stream)
        except Exception as e:  # secondary measurement; never fail the headline
            line["c5_sample"] = {"error": repr(e)}
    if world == 1 and not args.no_trace:
        try:
            line["trace"] = trace_measure(bb, torch, dev, stream)
        except Exception as e:  # secondary measurement; never fail the headline
            line["trace"] = {"error": repr(e)}
    if world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            req, secs = reference_sample(pts, args.ref_reps, threads)
            line["cpu_baseline"] = {
                "value": req / secs, "unit": "requests/s", "cores": threads, "kind": "reference",
                "sample": f"{len(pts)} C3 points x {args.ref_reps} replications x "
                          f"{args.requests} requests ({req} requests, {secs:.1f} s wall)"}
        except Exception as e:
            line["cpu_baseline"] = {"error": repr(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def c4_measure(bb, torch, stream, reps=12_500, n=100_000):
    """Secondary: BASELINE config 4 (noisy length predictor): k in {4, 8} x
    symmetric misassignment p_e in {0, 0.05, ..., 0.30}, B = 32, U[1, 20]
    lengths, lambda = 0.9 x the k-bin capacity, with exact per-replication
    quantiles; 10^5 replicas across 8 GPUs is 12,500 per GPU per point.  One
    shard launch per k (7 points), timed with CUDA events; the latency means
    must be non-decreasing in p_e (common random numbers across p_e)."""
    pes = [0.0, 0.05, 0.10, 0.15, 0.20, 0.25, 0.30]
    svc = bb.ServiceSpec("uniform", 1.0, 20.0)
    total_ms, monotone, per_k = 0.0, True, {}
    for k in (4, 8):
        lam = 0.9 * capacity(32, k, 1.0, 20.0)
        pts = [bb.RunTemplate(arrival_rate=lam, n_requests=n, batch_size=32, bins=bb.BinRule(k=k),
                              service=svc, error=bb.ErrorSpec("symmetric", pe)) for pe in pes]
        rep = torch.zeros(6 * reps * len(pts), dtype=torch.float64, device="cuda")
        bb.points_shard_device(pts, reps, 4, 0, reps, rep.data_ptr(), stream.cuda_stream)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bb.points_shard_device(pts, reps, 4, 0, reps, rep.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        res = bb.points_reduce_device(pts, reps, rep.data_ptr(), stream.cuda_stream)
        lat = [p.latency_mean for p in res]
        monotone &= all(b >= a for a, b in zip(lat, lat[1:]))
        per_k[f"k{k}"] = {"latency_mean": lat, "latency_p99": [p.latency_p99 for p in res]}
    req = 2 * len(pes) * reps * n
    return {"workload": f"C4 grid: k in {{4,8}} x p_e {pes} symmetric, B=32, U[1,20], lambda=0.9 cap, "
                        f"{reps} replications x {n} requests per point",
            "value": req / (total_ms / 1e3), "unit": "requests/s", "ms": total_ms,
            "latency_nondecreasing_in_p_e": monotone, **per_k}


def c5_measure(bb, torch, stream, reps=148 * 16 * 32, n=1_000_000):
    """Secondary: BASELINE config 5's shape (k=16, B=64, log-normal service
    exp(N(0,1)), 10^6 requests per replication) on a bounded sample of
    replications (one per resident thread of a full grid), lambda = 0.9 x the
    capacity of a pilot overload run.  With exact per-replication quantiles
    the request log (14 B/request) bounds how many 10^6-request replications
    run at once (HBM capacity), so this shape runs at a fraction of the
    sweep's rate; the quantiles-off figure is the A/B reference."""
    svc = bb.ServiceSpec("lognormal", mu=0.0, sigma=1.0)
    pilot = bb.run_point(bb.RunTemplate(n_requests=100_000, batch_size=64, bins=bb.BinRule(k=16),
                                        service=svc), 7, 512)
    lam = 0.9 * pilot.throughput_mean
    t = bb.RunTemplate(arrival_rate=lam, n_requests=n, batch_size=64, bins=bb.BinRule(k=16),
                       service=svc)
    rep = torch.zeros(6 * reps, dtype=torch.float64, device="cuda")
    out = {}
    for quant in (False, True):  # (the quantile run last: its p50/p99 are reported)
        prev = bb.set_generated_quantiles(quant)
        try:
            bb.points_shard_device([t], reps, 11, 0, reps, rep.data_ptr(), stream.cuda_stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            bb.points_shard_device([t], reps, 11, 0, reps, rep.data_ptr(), stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize()
            out[quant] = reps * n / (e0.elapsed_time(e1) / 1e3)
        finally:
            bb.set_generated_quantiles(prev)
    p = bb.points_reduce_device([t], reps, rep.data_ptr(), stream.cuda_stream)[0]
    return {"workload": f"C5 shape: k=16, B=64, lognormal(0,1) service, lambda=0.9 x pilot "
                        f"capacity ({lam:.4f}), {reps} replications x {n} requests",
            "value": out[True], "unit": "requests/s", "without_quantiles": out[False],
            "throughput_mean": p.throughput_mean, "latency_p50_mean": p.latency_p50,
            "latency_p99_mean": p.latency_p99}


def latest_profile(name):
    """profiles/r<NN>_<name> of the latest round that has it (ncu summaries)."""
    d = os.path.join(ROOT, "profiles")
    if not os.path.isdir(d):
        return None
    hits = sorted(f for f in os.listdir(d) if f.startswith("r") and f.endswith("_" + name))
    return os.path.join(d, hits[-1]) if hits else None


def trace_measure(bb, torch, dev, stream, n=10_000_000):
    """Secondary: BASELINE config 2 (10^7-request trace, k=8, B=16) in trace
    mode with the arrays resident in HBM -- the HBM-bound pipeline.

    The trace is produced by the unmodified reference (oracle/_ref, the
    checker): its run_simulation_detailed gives arrivals, services and
    predicted bins, and its batch finish times / metrics are what the
    device result is compared with (bit for bit).  Without the reference
    shim the streams come from the engine's host mt19937_64 streams and the
    check is reported as unavailable."""
    lam = 0.95 * capacity(16, 8, 1.0, 20.0)
    edges = bb.uniform_boundaries(8, 1.0, 20.0)
    ref = None
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle_py as O
        if O.have_reference():
            mr, dr = O.run(O.reference(), dict(arrival_rate=lam, n_requests=n, batch_size=16,
                                               edges=edges.edges, lo=1.0, hi=20.0, seed=1001,
                                               error="symmetric", p_error=0.1), detail=True)
            ref = (mr, dr)
    except Exception as e:  # the checker is optional; the measurement is not
        ref = None
        print(f"trace check: reference unavailable ({e!r})", file=sys.stderr)
    if ref is not None:
        a_h, s_h = ref[1]["req_arrival"], ref[1]["req_service"]
        p_h = ref[1]["req_pred_bin"].astype("uint8")
    else:
        cfg = bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=16, bins=edges,
                           service=bb.Uniform(1.0, 20.0), error_model=bb.Symmetric(0.1),
                           seed=1001, rng="reference")
        res = bb.run_simulation_detailed(cfg)
        a_h, s_h = res.requests["arrival"], res.requests["service"]
        p_h = res.requests["predicted_bin"]
    a = torch.from_numpy(a_h).to(dev)
    s = torch.from_numpy(s_h).to(dev)
    p = torch.from_numpy(p_h).to(dev)
    tcfg = bb.SimConfig(arrival_rate=lam, n_requests=n, batch_size=16, bins=edges)
    for _ in range(3):
        m = bb.run_trace_device(tcfg, a.data_ptr(), s.data_ptr(), 0, p.data_ptr(), stream.cuda_stream)
    times, parts = [], []
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        m = bb.run_trace_device(tcfg, a.data_ptr(), s.data_ptr(), 0, p.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        parts.append(bb.last_kernel_ms()[0])
    # end to end through the host-facing C ABI (bb_run_trace): the arrays start
    # in pinned host memory, the call uploads them (17 B/request), runs the
    # pipeline and returns the metrics to the host
    a_pin = torch.from_numpy(a_h).pin_memory()
    s_pin = torch.from_numpy(s_h).pin_memory()
    p_pin = torch.from_numpy(p_h).pin_memory()
    bb.run_trace(tcfg, a_pin.numpy(), s_pin.numpy(), pred_bin=p_pin.numpy())
    e2e_t = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bb.run_trace(tcfg, a_pin.numpy(), s_pin.numpy(), pred_bin=p_pin.numpy())
        e2e_t.append(time.perf_counter() - t0)
    te = sorted(e2e_t)[len(e2e_t) // 2]
    check = "reference unavailable"
    if ref is not None:  # after the timed runs: the device result vs the reference binary
        mr, dr = ref
        det = bb.run_trace(tcfg, a_h, s_h, pred_bin=p_h, detailed=True)
        fin = det.batches["finish_time"]
        same = (len(fin) == len(dr["bat_finish"])
                and bool((fin.view("uint64") == dr["bat_finish"].view("uint64")).all())
                and m.makespan == mr["makespan"] and m.latency_p50 == mr["latency_p50"]
                and m.latency_p99 == mr["latency_p99"] and m.n_completed == mr["n_completed"])
        check = "bit-exact" if same else "MISMATCH"
    t = sorted(times)[len(times) // 2]
    tp = sorted(parts)[len(parts) // 2]
    # partition kernel algorithmic bytes: read a,s (16) + pred (1); write pb (1) + rank (4)
    # + closing records (8+8+1+4+4 per batch = 25/B)
    part_bytes = n * (16 + 1 + 1 + 4) + (n / 16) * 25
    traffic = None  # DRAM bytes of one partition (its kernels), from one `ncu --set full` capture
    prof = latest_profile("trace_c2_ncu.json")
    if prof:
        caps = json.load(open(prof))
        parts_b = [c["dram_bytes_per_request"] for c in (caps if isinstance(caps, list) else [caps])
                   if c.get("dram_bytes_per_request") and any(
                       x in c.get("kernel", "") for x in ("partition_kernel", "count_kernel", "tscan_kernel",
                                                           "place_kernel"))]
        if parts_b:
            traffic = sum(parts_b) * n
    return {"workload": "C2: 10^7-request trace from the reference generator, k=8, B=16, "
                        "lambda=0.95 cap, Symmetric(0.1) predictions as input",
            "value": n / (t / 1e3), "unit": "requests/s", "ms_per_run": t,
            "vs_reference_binary": check,
            "e2e": {"value": n / te, "unit": "requests/s", "ms_per_run": te * 1e3,
                    "h2d_bytes_per_step": int(n * 17), "d2h_bytes_per_step": __import__("ctypes").sizeof(bb._capi.SimMetricsC),
                    "api": "bb_run_trace (pinned host arrays in, host metrics out)"},
            "roofline": {"bound": "hbm", "kernel": "partition (count_kernel + tscan_kernel + place_kernel)", "kernel_ms": tp,
                         "achieved": part_bytes / (tp / 1e3) / 1e9,
                         "peak": measured_peaks()["hbm_gbs"], "unit": "GB/s",
                         "frac": part_bytes / (tp / 1e3) / 1e9 / measured_peaks()["hbm_gbs"],
                         "traffic": traffic,
                         "algorithmic": "22 B/request + 25 B/batch (reads a,s,pred; writes bin, rank, records)"}}


if __name__ == "__main__":
    sys.exit(main())
