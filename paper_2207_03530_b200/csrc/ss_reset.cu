// ss_reset.cu — Env.reset / reset_at as device kernels with numpy's Philox
// stream (env.py:189-198 -> Scenario.reset_world_at -> common.scatter/place
// -> batching.uniform_in_box -> SeededRng.uniform).
//
// The reset program (SsResetOp) runs per env on a float32 register file;
// each draw instruction takes the next draw slot.  Whole-batch reset
// (reference reset()): every draw call covers the whole batch, x block then
// y block (batching.py:212-213), so env e (global index) reads draw
// slot*Bg + e.  Masked reset: identical to calling reset(env_index=i) for each
// selected i in ascending order; the env of rank r among the selected reads
// draw r*n_slots + slot.  The rank is a prefix count over the mask (count ->
// scan -> apply), with an optional per-shard base so a sharded run
// reproduces the single-GPU stream bitwise.
#include "ss_internal.cuh"

namespace ss {

constexpr int kResetThreads = 256;

struct ResetArgs {
  DevState s;
  const SsEntityDesc* ents;
  const SsResetOp* ops;
  int n_ops;
  int n_slots;
  int n_flag_words;
  const uint8_t* mask;        // nullptr: whole batch
  const int64_t* block_off;   // masked: exclusive prefix of selected envs per block (+ base)
};

SS_DEV void set_pos(const DevState& s, const SsEntityDesc& d, int64_t e, float x, float y) {
  if (d.movable) {
    float4* q = s.dyn + d.slot * s.B + e;
    float4 v = *q;
    v.x = x; v.y = y;
    *q = v;
  } else {
    s.stat[d.slot * s.B + e] = make_float2(x, y);
  }
}

SS_DEV void zero_motion(const DevState& s, const SsEntityDesc& d, int k, int64_t e) {
  if (d.movable) {
    float4* q = s.dyn + d.slot * s.B + e;
    float4 v = *q;
    v.z = 0.0f; v.w = 0.0f;
    *q = v;
  } else {
    s.stat_vel[d.slot * s.B + e] = make_float2(0.0f, 0.0f);
  }
  reinterpret_cast<float*>(s.rot)[2 * (k * s.B + e) + 1] = 0.0f;   // ang_vel; rot kept
}

// Run the reset program for env e.  draw(slot) yields the slot's 64-bit draw.
template <class Draw>
SS_DEV void reset_env(const ResetArgs& a, int64_t e, Draw draw) {
  const int64_t B = a.s.B;
  float R[SS_RESET_REGS];
  int slot = 0;
  for (int j = 0; j < a.n_ops; ++j) {
    const SsResetOp op = a.ops[j];
    switch (op.kind) {
      case SS_RESET_SCATTER:
      case SS_RESET_PLACE: {
        float x, y;
        if (op.kind == SS_RESET_SCATTER) {
          x = uniform_f32(draw(slot), op.lo_x, op.range_x);
          y = uniform_f32(draw(slot + 1), op.lo_y, op.range_y);
          slot += 2;
        } else {
          x = (float)op.lo_x;
          y = (float)op.lo_y;
        }
        const SsEntityDesc& d = a.ents[op.entity];
        set_pos(a.s, d, e, x, y);
        zero_motion(a.s, d, op.entity, e);
        break;
      }
      case SS_RESET_DRAW: R[op.r0] = uniform_f32(draw(slot++), op.lo_x, op.range_x); break;
      case SS_RESET_CONST: R[op.r0] = (float)op.lo_x; break;
      case SS_RESET_ADD: R[op.r0] = fadd(R[op.r1], R[op.r2]); break;
      case SS_RESET_NEG: R[op.r0] = -R[op.r1]; break;
      case SS_RESET_LOADPOS: {
        const SsEntityDesc& d = a.ents[op.entity];
        float v;
        if (d.movable) { const float4 q = a.s.dyn[d.slot * B + e]; v = op.axis ? q.y : q.x; }
        else { const float2 q = a.s.stat[d.slot * B + e]; v = op.axis ? q.y : q.x; }
        R[op.r0] = v;
        break;
      }
      case SS_RESET_SETPOS: set_pos(a.s, a.ents[op.entity], e, R[op.r0], R[op.r1]); break;
      case SS_RESET_SETROT: reinterpret_cast<float*>(a.s.rot)[2 * (op.entity * B + e)] = R[op.r0]; break;
      case SS_RESET_ZERO: zero_motion(a.s, a.ents[op.entity], op.entity, e); break;
      default: break;
    }
  }
  a.s.step_count[e] = 0;
  for (int w = 0; w < a.n_flag_words; ++w) a.s.flags[w * B + e] = 0u;
  if (a.s.aux) a.s.aux[e] = 0.0f;
}

__global__ void __launch_bounds__(kResetThreads) k_reset_all(const ResetArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    philox_advance(a.s.rng_in, (uint64_t)a.n_slots * (uint64_t)a.s.global_batch, a.s.rng_out);
  }
  if (e >= a.s.B) return;
  const uint64_t eg = (uint64_t)(a.s.env_offset + e);
  const uint64_t Bg = (uint64_t)a.s.global_batch;
  reset_env(a, e, [&](int slot) { return philox_draw(a.s.rng_in, (uint64_t)slot * Bg + eg); });
}

// Per-block selected counts.
__global__ void __launch_bounds__(kResetThreads) k_mask_count(const uint8_t* mask, int64_t B,
                                                              int64_t* block_cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int sel = (e < B) && mask[e];
  const int c = __syncthreads_count(sel);
  if (threadIdx.x == 0) block_cnt[blockIdx.x] = c;
}

// Exclusive scan of the block counts (one CTA), the shard total, and the
// advanced RNG state (total over all shards * draws per env).
__global__ void __launch_bounds__(1024) k_mask_scan(int64_t* block_cnt, int nblocks,
                                                     const int64_t* base, const int64_t* total,
                                                     uint64_t draws_per_env, const uint64_t* rng_in,
                                                     uint64_t* rng_out, int64_t* local_total) {
  __shared__ int64_t warp_sums[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = base ? *base : 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int off = 0; off < nblocks; off += 1024) {
    const int i = off + threadIdx.x;
    const int64_t v = i < nblocks ? block_cnt[i] : 0;
    int64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int64_t w = warp_sums[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += y;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int64_t incl = x + (wid > 0 ? warp_sums[wid - 1] : 0);
    if (i < nblocks) block_cnt[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int64_t local = carry - (base ? *base : 0);
    if (local_total) *local_total = local;
    const int64_t tot = total ? *total : local;
    if (rng_out) philox_advance(rng_in, (uint64_t)tot * draws_per_env, rng_out);
  }
}

__global__ void __launch_bounds__(kResetThreads) k_reset_masked(const ResetArgs a) {
  __shared__ int warp_cnt[kResetThreads / 32];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool sel = (e < a.s.B) && a.mask[e];
  const unsigned bal = __ballot_sync(0xffffffffu, sel);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) warp_cnt[wid] = __popc(bal);
  __syncthreads();
  if (!sel) return;
  int before = 0;
  for (int w = 0; w < wid; ++w) before += warp_cnt[w];
  before += __popc(bal & ((1u << lane) - 1u));
  const uint64_t rank = (uint64_t)(a.block_off[blockIdx.x] + before);
  const uint64_t per = (uint64_t)a.n_slots;
  reset_env(a, e, [&](int slot) { return philox_draw(a.s.rng_in, rank * per + (uint64_t)slot); });
}

int launch_reset(World& w, const SsBuffers* buf, const uint8_t* mask, const int64_t* mask_base,
                 const int64_t* mask_total, cudaStream_t st) {
  ResetArgs a;
  memset(&a, 0, sizeof(a));
  a.s = make_state(w, buf);
  a.ents = w.d_ents;
  a.ops = w.d_reset_ops;
  a.n_ops = (int)w.reset_ops.size();
  a.n_slots = w.n_slots;
  a.n_flag_words = w.d.n_flag_words;
  const int64_t B = w.d.batch;
  const unsigned grid = (unsigned)((B + kResetThreads - 1) / kResetThreads);
  if (mask == nullptr) {
    k_reset_all<<<grid, kResetThreads, 0, st>>>(a);
    return cuda_status(cudaGetLastError(), "reset launch");
  }
  if ((int64_t)grid + 1 > w.scan_cap) {
    set_error("reset scratch too small");
    return SS_ERR_CUDA;
  }
  k_mask_count<<<grid, kResetThreads, 0, st>>>(mask, B, w.d_scan);
  k_mask_scan<<<1, 1024, 0, st>>>(w.d_scan, (int)grid, mask_base, mask_total,
                                  (uint64_t)w.n_slots, a.s.rng_in, a.s.rng_out,
                                  w.d_scan + grid);
  a.mask = mask;
  a.block_off = w.d_scan;
  k_reset_masked<<<grid, kResetThreads, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "masked reset launch");
}

int launch_mask_count(World& w, const uint8_t* mask, int64_t* count_out, cudaStream_t st) {
  const int64_t B = w.d.batch;
  const unsigned grid = (unsigned)((B + kResetThreads - 1) / kResetThreads);
  if ((int64_t)grid + 1 > w.scan_cap) { set_error("reset scratch too small"); return SS_ERR_CUDA; }
  k_mask_count<<<grid, kResetThreads, 0, st>>>(mask, B, w.d_scan);
  k_mask_scan<<<1, 1024, 0, st>>>(w.d_scan, (int)grid, nullptr, nullptr, 0, nullptr, nullptr,
                                  count_out);
  return cuda_status(cudaGetLastError(), "mask count launch");
}

}  // namespace ss
