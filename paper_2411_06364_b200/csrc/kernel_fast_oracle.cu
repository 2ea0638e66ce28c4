// kernel_fast_oracle.cu — kernel_fast.cu specialised one step further for
// econoserve-full with the oracle predictor (ECONO_SPEC_ORACLE_FULL: the
// noisy predictors' code — normal draws, glibc exp/log, Lemire draws — and
// the non-pipelining branch drop out; 16.9k instructions against 20.0k).
// Launched when every econoserve instance of the batch is that configuration
// (BASELINE configs[0]-[2]); same results as the other step kernels.
#define ECONO_SPEC_ORACLE_FULL 1
#define FAST_KERNEL k_engine_steps_fast_oracle
#define FAST_LAUNCH launch_engine_steps_fast_oracle
#include "kernel_fast.cu"
