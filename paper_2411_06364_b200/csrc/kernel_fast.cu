// kernel_fast.cu — the econoserve step kernel specialised at compile time for
// the common serving configuration: no event/sample recording (ECONO_NOREC:
// REC_EV / REC_SM constant false) and the ordered PT queue
// (ECONO_SPEC_ORDERED: the FIFO min-tree paths drop out). The code the warps
// execute is smaller and denser in the instruction cache (ncu: 38% of stall
// samples are instruction fetch). econo_batch launches it when every
// econoserve instance of the batch records nothing and orders its PT queue
// (econoserve-sdo/-full; the bench path); the results are those of
// k_engine_steps for the same batch.
#define ECONO_NOREC 1
#define ECONO_SPEC_ORDERED 1
#ifndef FAST_KERNEL  // kernel_fast_oracle.cu includes this file with its own names
#define FAST_KERNEL k_engine_steps_fast
#define FAST_LAUNCH launch_engine_steps_fast
#endif
#include "steps.cuh"

#include <cuda_runtime.h>

using namespace econo;

__global__ void __launch_bounds__(32) FAST_KERNEL(Inst* insts, int64_t max_steps, int64_t slice_ns) {
  if (insts[blockIdx.x].base) return;  // a baseline-policy instance (k_baseline_steps)
  const int64_t deadline = slice_ns > 0 ? now_ns() + slice_ns : 0;
  __shared__ Inst I;
  const int64_t t0 = PROF_NOW();
  inst_load(I, &insts[blockIdx.x]);
  engine_steps<false>(I, steps_for(I, max_steps), deadline);
  LANE0(I.prof[11] += PROF_NOW() - t0; I.prof[12]++);
  inst_store(&insts[blockIdx.x], I);
}

void FAST_LAUNCH(Inst* insts, unsigned n_inst, int64_t max_steps, int64_t slice_ns, cudaStream_t s) {
  FAST_KERNEL<<<n_inst, 32, 0, s>>>(insts, max_steps, slice_ns);
}
