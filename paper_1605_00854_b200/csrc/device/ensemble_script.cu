// Scripted-replay build of the sub-warp trajectory kernel: the same kernel
// source as ensemble.cu with the stream's draw blocks read from a
// caller-supplied script (dev_run_params::script_hi / script_lo) instead of
// Philox. Serves pbn_gpu_run_scripted — the device counterpart of the
// reference tests' scripted_rng (tests/oracles.hpp:235-254,
// test_engine.cpp:89-153). A separate translation unit so that the production
// kernels' code generation is untouched.
#define PBN_SCRIPT_TU 1
#include "ensemble.cu"
