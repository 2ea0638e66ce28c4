// steps.cuh — the per-instance step loop (Engine::run()'s body) and the
// shared-memory staging of an instance, shared by the two translation units
// that instantiate the step kernel: runtime.cu (every configuration) and
// kernel_fast.cu (specialised at compile time: no recording, ordered PT queue).
#pragma once
#include "engine.cuh"

namespace econo {

// Engine::run()'s loop body, up to max_steps times (engine.hpp:118-122).
// The quiet-span test is only worth running after a normal step that
// completed nothing: a replay always stops right before an event step (or at
// the budget), and a step after a completion finds freed KVC for the GT
// queue head. Skipping the test is always exact — it only decides whether a
// replay may stand in for normal steps.
// Device wall clock (ns), for time-sliced launches. Read by lane 0 and
// broadcast, so every break decision taken on it is warp-uniform by
// construction (the step body's full-mask shuffles and ballots need that).
// Call from warp-converged code only.
EDEV int64_t now_ns() {
#ifdef __CUDA_ARCH__
  uint64_t t;  // every lane reads (no divergent branch); lane 0's value is the one used
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (int64_t)__shfl_sync(0xffffffffu, t, 0);
#else
  return 0;
#endif
}

// max_steps < 0 encodes an absolute target (econo_batch_launch_to): advance
// until Engine::step() has been called -max_steps times in total.
EDEV int64_t steps_for(const Inst& I, int64_t max_steps) {
  return max_steps >= 0 ? max_steps : (-max_steps > I.steps ? -max_steps - I.steps : 0);
}

// deadline_ns > 0 (a time-sliced launch, econo_batch_launch_slice): stop at
// the first step boundary past the deadline; every instance then advances as
// far as the slice allows instead of all waiting for the slowest one.
template <bool B>
EDEVNI void engine_steps(Inst& I, int64_t max_steps, int64_t deadline_ns = 0) {
  LANE0(I.status = STATUS_RUN);
  bool test = true;
  for (int64_t s = 0; s < max_steps;) {
    if (I.error || I.completed >= I.n) break;
    if (deadline_ns && now_ns() >= deadline_ns) break;
    if ((REC_EV(I) && I.ev_n + step_event_bound(I) > I.ev_cap) ||
        (REC_SM(I) && I.sm_n + 1 > I.sm_cap)) {
      LANE0(I.status = STATUS_DRAIN);
      break;
    }
    if (!B && I.skip && test) {
      const int64_t t0 = PROF_NOW();
      bool fuse = false;
      const int64_t k = quiet_span(I, max_steps - s, &fuse);
      const int64_t t1 = PROF_NOW();
      UNI(I.prof[0] += t1 - t0);  // counters: any lane's clock delta will do (no divergence)
      if (k > 0 || fuse) {
        s += quiet_steps(I, k, fuse);
        UNI(I.prof[1] += PROF_NOW() - t1; I.prof[4]++);
        test = false;
        continue;
      }
    }
    const int64_t t2 = PROF_NOW();
    const int64_t c0 = I.completed;
    engine_step<B>(I);
    UNI(I.prof[2] += PROF_NOW() - t2; I.prof[5]++);
    test = I.completed == c0;
    ++s;
  }
}

}  // namespace econo

#if defined(__CUDACC__) && !defined(ECONO_HOSTSIM)
using econo::Inst;
// Inst staged in shared memory for the launch; one warp per instance.
__device__ __forceinline__ void inst_load(Inst& s, const Inst* g) {
  const uint64_t* src = reinterpret_cast<const uint64_t*>(g);
  uint64_t* dst = reinterpret_cast<uint64_t*>(&s);
  for (int i = threadIdx.x; i < (int)(sizeof(Inst) / 8); i += 32) dst[i] = src[i];
  __syncwarp();
}
__device__ __forceinline__ void inst_store(Inst* g, const Inst& s) {
  __syncwarp();
  const uint64_t* src = reinterpret_cast<const uint64_t*>(&s);
  uint64_t* dst = reinterpret_cast<uint64_t*>(g);
  for (int i = threadIdx.x; i < (int)(sizeof(Inst) / 8); i += 32) dst[i] = src[i];
}

#endif
