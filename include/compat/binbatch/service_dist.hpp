#pragma once
// Drop-in forwarding header: the reference's "binbatch/service_dist.hpp" name resolves
// to the B200 engine's C++ API.  Put include/compat first on the include
// path, leave the reference program unchanged, link libbinbatch_b200.so.
#include "../../binbatch_b200/binbatch.hpp"
