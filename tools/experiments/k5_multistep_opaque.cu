// EXPERIMENT (not product): K5's interpreter with the multi-step loop inside one launch, the state in
// registers, and the phase dispatch compiled the natural way (no opaque() copies).  Built by
// tools/experiments/k5_multistep.py at several optimisation levels to isolate the round-1 report
// ("lost whole warps' stores after ~10 steps at -O3").
#include "common.cuh"
namespace {

enum Phase : int { AwaitGoal = 0, Goal = 1, Wait = 2, AwaitConclusionTag = 3, Conclusion = 4, AwaitClose = 5 };
enum Tag : int {
  ParallelOpen = 0, ParallelClose, GoalOpen, GoalClose, OutlineOpen, OutlineClose, PathOpen, PathClose,
  ConclusionOpen, ConclusionClose
};

struct Act {
  int kind, arg;
};

__device__ __forceinline__ Act violation(int code) { return {MV_ACT_VIOLATION, code}; }

// An opaque copy: each phase test compares a value the compiler cannot prove equal to the
// others, so the chain is not folded back into a jump table (see feed()).
__device__ __forceinline__ int opaque(int x) {
  int y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// One event on one lane (engine.cpp:323-415). Violations leave the state untouched, as there.
__device__ __forceinline__ Act feed(int32_t* st, int ev) {
  const int depth = st[0] & 0xff;
  const bool child = (st[0] >> 8) & 1;
  if (ev == MV_INTERP_IDLE) return {MV_ACT_NONE, 0};
  if (ev == MV_INTERP_MERGED) {  // engine.cpp:793
    if (depth == 0) return violation(MV_VIOL_MERGE_NO_BLOCK);
    st[1] = (st[1] & ~7) | AwaitConclusionTag;
    return {MV_ACT_NONE, 0};
  }
  const bool is_tag = ev >= 0 && ev < 10;
  if (depth == 0) {  // engine.cpp:332-349
    if (!is_tag) return {MV_ACT_NONE, 0};
    if (ev == ParallelOpen) {
      st[1] = AwaitGoal;
      st[0] = 1 | (child << 8);
      return {MV_ACT_NONE, 0};
    }
    if (ev == PathOpen && child) return {MV_ACT_NONE, 0};  // BUG-2 fix (oracle/ref_patch.py)
    if (ev == PathClose) return child ? Act{MV_ACT_WORKER_DONE, 0} : violation(MV_VIOL_PATH_CLOSE_OUTSIDE);
    return violation(MV_VIOL_UNEXPECTED_SEQUENTIAL);
  }
  const int f = st[1];
  const int phase = f & 7;
  const bool in_outline = (f >> 3) & 1, after_outline = (f >> 4) & 1;
  // An if-chain over opaque copies, not a switch.  Root cause (tools/experiments/k5_multistep.py,
  // B200, CUDA 12.9.86): ptxas lowers a switch or a plain if-chain over the phase to a jump table
  // (`LDC c[0x2][idx]` + `BRX`); when the lanes of a warp sit in different phases that indirect
  // branch is divergent, and every build that contains it (ptxas -O1 and -O3; one step per launch
  // or a multi-step loop) corrupts the launch — illegal memory accesses, or, in round 1's variant,
  // whole warps' stores lost — while the same PTX compiled without the jump table (ptxas -O0, -G)
  // is exact, and the jump-table build is exact when all lanes share one phase.  opaque() hides
  // the equality chain from that lowering: the SASS has compares and predicated branches only.
  if (opaque(phase) == AwaitGoal) {
    if (ev != GoalOpen) return violation(MV_VIOL_EXPECTED_GOAL);
    st[1] = (f & ~7) | Goal;
    return {MV_ACT_NONE, 0};
  }
  if (opaque(phase) == Goal) {
    if (!is_tag) return (after_outline && !in_outline) ? violation(MV_VIOL_TEXT_BETWEEN_OUTLINES) : Act{0, 0};
    if (ev == OutlineOpen) {
      if (in_outline) return violation(MV_VIOL_NESTED_OUTLINE);
      st[1] = (f | 8) + 256;  // in_outline, ++outlines
      return {MV_ACT_NONE, 0};
    }
    if (ev == OutlineClose) {
      if (!in_outline) return violation(MV_VIOL_OUTLINE_CLOSE_WITHOUT_OPEN);
      st[1] = (f & ~8) | 16;
      return {MV_ACT_NONE, 0};
    }
    if (ev == GoalClose) {
      if (in_outline) return violation(MV_VIOL_GOAL_CLOSE_IN_OUTLINE);
      if ((f >> 8) == 0) return violation(MV_VIOL_ZERO_OUTLINES);
      st[1] = (f & ~7) | Wait;
      return {MV_ACT_SPAWN, f >> 8};
    }
    return violation(MV_VIOL_UNEXPECTED_IN_GOAL);
  }
  if (opaque(phase) == Wait) return violation(MV_VIOL_WAITING);
  if (opaque(phase) == AwaitConclusionTag) {
    if (ev != ConclusionOpen) return violation(MV_VIOL_EXPECTED_CONCLUSION);
    st[1] = (f & ~7) | Conclusion;
    return {MV_ACT_NONE, 0};
  }
  if (opaque(phase) == Conclusion) {
    if (!is_tag) return {MV_ACT_NONE, 0};
    if (ev != ConclusionClose) return violation(MV_VIOL_UNEXPECTED_IN_CONCLUSION);
    st[1] = (f & ~7) | AwaitClose;
    return {MV_ACT_NONE, 0};
  }
  // AwaitClose
  if (ev != ParallelClose) return violation(MV_VIOL_EXPECTED_PARALLEL_CLOSE);
  st[0] = (depth - 1) | (child << 8);
  return {MV_ACT_NONE, 0};
}

}  // namespace

__global__ void interp_multi_kernel(int32_t* __restrict__ state, int32_t n_lanes, const int32_t* __restrict__ events,
                                    int32_t n_steps, int32_t* __restrict__ action, int32_t* __restrict__ arg) {
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  if (lane >= n_lanes) return;
  int32_t st[MV_INTERP_STATE_WORDS];
#pragma unroll
  for (int w = 0; w < MV_INTERP_STATE_WORDS; ++w) st[w] = state[(int64_t)lane * MV_INTERP_STATE_WORDS + w];
  for (int s = 0; s < n_steps; ++s) {
    const int64_t i = (int64_t)s * n_lanes + lane;
    const Act a = feed(st, events[i]);
    action[i] = a.kind;
    arg[i] = a.arg;
  }
#pragma unroll
  for (int w = 0; w < MV_INTERP_STATE_WORDS; ++w) state[(int64_t)lane * MV_INTERP_STATE_WORDS + w] = st[w];
}

extern "C" MV_API int k5x_run(int32_t* d_state, int32_t n_lanes, const int32_t* d_events, int32_t n_steps,
                              int32_t* d_action, int32_t* d_arg) {
  interp_multi_kernel<<<(n_lanes + 127) / 128, 128>>>(d_state, n_lanes, d_events, n_steps, d_action, d_arg);
  return (int)cudaDeviceSynchronize();
}
