// K5 — per-lane tag interpreter on the device.
//
// Restates the engine's runtime counting rule, feed_interpreter (engine.cpp:323-415, with the
// BUG-2 fix: a worker lane accepts its injected <Path>), plus the merge completion that resets
// the top frame to AwaitConclusionTag (engine.cpp:793), for every lane of every request in one
// launch: the decode step's sampled token ids stay on the device, and the Map trigger
// (</Goal> -> spawn count = outlines), WorkerDone (</Path>) and grammar violations come back as
// per-lane actions plus a compacted spawn list a fork launch can consume.
//
// Lane state is caller-owned: MV_INTERP_STATE_WORDS (2) int32 per lane, word 0 = depth |
// is_child << 8, word 1 = the frame (InterpFrame, engine.cpp:279-285) packed as phase |
// in_outline << 3 | after_outline << 4 | outlines << 8. The reference's frame vector never holds
// more than one frame: it pushes only when empty (engine.cpp:335-337) and a <Parallel> anywhere
// else is a violation; nested blocks live on the worker lanes' own stacks.
// One thread per lane and one launch per step (see interp_kernel); lanes are independent. The work is a
// few dozen bytes per lane per step (latency-bound, not a roofline kernel).
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
  // An if-chain over opaque copies, not a switch, and one step per launch (interp_kernel): the two
  // conditions under which this code is exact on B200 with CUDA 12.9.86.  Measured with the same
  // PTX built several ways (tools/experiments/k5_multistep.py, 16K random lanes x 48 steps against
  // the restatement): with warp-divergent per-lane phases, every ptxas-optimised build (-O1, -O3)
  // of the plain dispatch (lowered to an `LDC c[0x2]` jump table + BRX) faults with an illegal
  // memory access, even at one step per launch; the opaque dispatch (compares only) faults inside
  // a multi-step loop; the same PTX compiled with ptxas -O0 or -G is exact in every form, and the
  // optimised builds are exact when all lanes share one phase.  The SASS of the failing loop shows
  // no out-of-range address arithmetic, so this is treated as a ptxas code-generation defect
  // around divergent reconvergence, not a source-level race (each lane owns its state and outputs).
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

// One decode step per launch (step index `step` for the spawn list): the engine's use, one sampled
// token per lane per step.  (A multi-step loop is correct too once the phase dispatch avoids the
// divergent jump table, see feed(); one launch per step keeps the spawn list ordered by step.)
__global__ void interp_kernel(int32_t* __restrict__ state, int32_t n_lanes, const int32_t* __restrict__ events,
                              int32_t step, int32_t* __restrict__ action, int32_t* __restrict__ arg,
                              int32_t* __restrict__ spawns, int32_t* __restrict__ n_spawns) {
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  if (lane >= n_lanes) return;
  int32_t st[MV_INTERP_STATE_WORDS];
#pragma unroll
  for (int w = 0; w < MV_INTERP_STATE_WORDS; ++w) st[w] = state[(int64_t)lane * MV_INTERP_STATE_WORDS + w];
  {
    const int s = step;
    const int64_t i = lane;  // this step's [lane] row: coalesced across the warp
    const int ev = events[i];
    const Act a = feed(st, ev);
    action[i] = a.kind;
    arg[i] = a.arg;
    if (a.kind == MV_ACT_SPAWN && spawns != nullptr) {
      const int slot = atomicAdd(n_spawns, 1);
      spawns[3 * slot] = s;
      spawns[3 * slot + 1] = lane;
      spawns[3 * slot + 2] = a.arg;
    }
  }
#pragma unroll
  for (int w = 0; w < MV_INTERP_STATE_WORDS; ++w) state[(int64_t)lane * MV_INTERP_STATE_WORDS + w] = st[w];
}

__global__ void interp_init_kernel(int32_t* __restrict__ state, int32_t n_lanes, const int32_t* __restrict__ is_child) {
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  if (lane >= n_lanes) return;
  state[(int64_t)lane * MV_INTERP_STATE_WORDS] = (is_child != nullptr && is_child[lane]) ? (1 << 8) : 0;
  for (int w = 1; w < MV_INTERP_STATE_WORDS; ++w) state[(int64_t)lane * MV_INTERP_STATE_WORDS + w] = 0;
}

using mv::fail;

extern "C" mv_status mv_interp_init(int32_t* d_state, int32_t n_lanes, const int32_t* d_is_child, mv_stream_t stream) {
  if (n_lanes < 0 || (n_lanes > 0 && d_state == nullptr))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_interp_init: bad arguments");
  if (n_lanes == 0) return MV_OK;
  interp_init_kernel<<<(n_lanes + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(d_state, n_lanes,
                                                                                                d_is_child);
  MV_LAUNCH_CHECK();
  return MV_OK;
}

extern "C" mv_status mv_interp_feed(int32_t* d_state, int32_t n_lanes, const int32_t* d_events, int32_t n_steps,
                                    int32_t* d_action, int32_t* d_arg, int32_t* d_spawns, int32_t* d_n_spawns,
                                    mv_stream_t stream) {
  if (n_lanes < 0 || n_steps < 0 || (d_spawns != nullptr && d_n_spawns == nullptr))
    return fail(MV_ERR_INVALID_ARGUMENT, "mv_interp_feed: bad arguments");
  if (n_lanes == 0 || n_steps == 0) return MV_OK;
  if (!d_state || !d_events || !d_action || !d_arg) return fail(MV_ERR_INVALID_ARGUMENT, "mv_interp_feed: null buffer");
  // 128-thread blocks: at a few hundred lanes per step this still spreads over many SMs
  for (int s = 0; s < n_steps; ++s) {
    const int64_t off = (int64_t)s * n_lanes;
    interp_kernel<<<(n_lanes + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        d_state, n_lanes, d_events + off, s, d_action + off, d_arg + off, d_spawns, d_n_spawns);
    MV_LAUNCH_CHECK();
  }
  return MV_OK;
}
