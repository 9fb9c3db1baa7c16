// ss_small.cuh — shared pieces of the thread-per-env fused step kernels
// (simple_spread, transport, dropout: ss_spread.cu / ss_transport.cu; the
// line / box catalog tasks: ss_catalog.cu; flocking: ss_flocking.cu): one
// thread per environment, the whole entity state of an env in registers for
// the duration of the step.
//
// One launch does, per env (env.py:209-235 order):
//   decode (env.py:97) -> forces: action, gravity, pair contacts in the
//   reference's lexicographic pair order (dynamics.py:151-180) -> integrate
//   (dynamics.py:182-184) -> post_step -> step_count += 1 -> rewards ->
//   done | horizon -> observations.
// HBM traffic: every state row read once and written once (float4 SoA rows,
// env index contiguous, so each warp access is a contiguous 512 B), actions
// read once, obs/reward/done written once (obs staged per warp in shared
// memory and streamed out with 16-byte stores).
//
// Each kernel family lives in its own translation unit (parallel builds) and
// exports a host launcher taking the SmallArgs that launch_small (ss_small.cu)
// fills from the world descriptor.
#pragma once
#include <cstdlib>

#include "ss_bulk.cuh"
#include "ss_physics.cuh"    // (includes ss_geometry.cuh, ss_internal.cuh)

namespace ss {

constexpr int kSmallMaxAgents = 8;
constexpr int kFlockMaxRocks = 6;
constexpr int kSmallThreads = 128;
// minimum resident CTAs per SM requested from ptxas (register budget)
#ifndef SS_SMALL_MINB
#define SS_SMALL_MINB 6   // 6 x 128 threads: <= 80 registers, best measured (tools/sweep_variants.py)
#endif

// Entity / pair descriptors the fixed-template kernels (simple_spread,
// transport) read by value from the kernel parameters: constant-bank
// operands of the arithmetic, no loads (and no registers waiting on them)
// inside the step.  SS_CONST_DESC=0 reads them from global memory instead.
#ifndef SS_CONST_DESC
#define SS_CONST_DESC 1
#endif
constexpr int kSmallConstEnts = kSmallMaxAgents + 1;                              // transport: + package
constexpr int kSmallConstPairs = kSmallMaxAgents * (kSmallMaxAgents - 1) / 2 + kSmallMaxAgents;

struct SmallArgs {
  DevState s;
  PhysK ph;
  const SsEntityDesc* ents;
  const SsPairDesc* pairs;
  const float2* act[kSmallMaxAgents];
  float* obs;
  int64_t obs_stride;   // floats between agent blocks
  float* rew;
  uint8_t* done;
  int mode;
  int raw_forces;
  int obs_dim;
  int E, P;             // entities, pairs (catalog kernels' in-launch world_step)
  int acc_off;          // floats of dynamic smem before its force accumulators
  int64_t e_begin;      // first env handled by this launch (tail launches)
  const int* guard;
  int guard_n;          // guard words to OR (SsStepIO.guard_count, >= 1)
  float sc[16];
  double sd[8];
  int si[8];
  // lidar (flocking extension)
  int n_rays;
  double lidar_range;
  double ray_start, ray_span;
  int attach_rot;
  const double* ray_dir;  // [n_rays][2] cos/sin of the base angles (numpy values)
  SsEntityDesc ek[kSmallConstEnts];   // ents[0 .. kSmallConstEnts) by value
  SsPairDesc pk[kSmallConstPairs];    // pairs[0 .. kSmallConstPairs) by value
};

// Descriptor i / pair p of a fixed-template kernel (compile-time index
// below the by-value counts).
SS_DEV const SsEntityDesc& tmpl_ent(const SmallArgs& a, int i) { return SS_CONST_DESC ? a.ek[i] : a.ents[i]; }
SS_DEV const SsPairDesc& tmpl_pair(const SmallArgs& a, int p) { return SS_CONST_DESC ? a.pk[p] : a.pairs[p]; }

// Flush one agent's staged obs rows (warp-private smem) to global memory.
SS_DEV void warp_flush(float* __restrict__ dst, int nvalid, int O, float* __restrict__ sbuf) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const int n = nvalid * O;
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) != 0) {
    for (int i = lane; i < n; i += 32) __stcs(dst + i, sbuf[i]);
    __syncwarp();
    return;
  }
  const int n4 = n >> 2;
  float4* d4 = reinterpret_cast<float4*>(dst);
  const float4* s4 = reinterpret_cast<const float4*>(sbuf);
  for (int i = lane; i < n4; i += 32) __stcs(d4 + i, s4[i]);
  for (int i = (n4 << 2) + lane; i < n; i += 32) __stcs(dst + i, sbuf[i]);
  __syncwarp();
}

// Observation flush through the bulk-copy engine (SS_OBS_BULK): each agent's
// 32 staged rows have their own staging block, so a full, 16-byte aligned
// warp block leaves with ONE cp.async.bulk store issued by lane 0 (the LSU
// and the other lanes are free at once); partial blocks take warp_flush.
// obs_bulk_drain() must run before the kernel exits (smem is read async).
#ifndef SS_OBS_BULK
#define SS_OBS_BULK 1   // measured: transport 1M envs 128 -> 118 us, simple_spread 59.3 -> 58.6 us
#endif
constexpr int kObsBulk = SS_OBS_BULK;

SS_DEV void warp_flush_bulk(float* __restrict__ dst, int nvalid, int O, float* __restrict__ sbuf) {
  const uint32_t bytes = (uint32_t)(nvalid * O) * 4u;
  if (nvalid == 32 && (bytes & 15u) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
    fence_proxy_async_smem();      // this lane's row -> visible to the async proxy
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      bulk_store(dst, sbuf, bytes);
      bulk_commit();
    }
    return;
  }
  warp_flush(dst, nvalid, O, sbuf);
}

SS_DEV void obs_bulk_drain() {
  if (kObsBulk && (threadIdx.x & 31) == 0) bulk_wait_read_all();
}

// Bulk flush when the per-agent staging blocks fit the default 48 KB of
// dynamic shared memory (every BASELINE config does); otherwise one block per
// warp, reused agent after agent.
__host__ __device__ constexpr bool obs_bulk(int NA, int O) { return kObsBulk && NA * O <= 96; }

// Staging buffers per warp for the bulk flush: one per agent, or a ring of
// SS_OBS_NBUF (a buffer is reused once its previous bulk store has read it).
#ifndef SS_OBS_NBUF
#define SS_OBS_NBUF 0     // 0: one per agent
#endif
__host__ __device__ constexpr int obs_nbuf(int NA, int O) {
  return !obs_bulk(NA, O) ? 1 : (SS_OBS_NBUF > 0 && SS_OBS_NBUF < NA ? SS_OBS_NBUF : NA);
}

// The warp's whole staging region (obs_nbuf blocks of 32 * O floats).
SS_DEV float* obs_stage_base(float* smem, int NA, int O) {
  return smem + (threadIdx.x >> 5) * obs_nbuf(NA, O) * (32 * O);
}

// Staging block of (warp, agent i).
SS_DEV float* obs_stage(float* smem, int i, int NA, int O) {
  const int nb = obs_nbuf(NA, O);
  if (obs_bulk(NA, O) && nb < NA && i >= nb) {
    // ring: the store issued nb agents ago must have read this buffer
    if ((threadIdx.x & 31) == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(SS_OBS_NBUF > 0 ? SS_OBS_NBUF - 1 : 0) : "memory");
    __syncwarp();
  }
  return smem + ((threadIdx.x >> 5) * nb + (i % nb)) * (32 * O);
}

SS_DEV void obs_flush(float* __restrict__ dst, int nvalid, int NA, int O, float* __restrict__ sbuf) {
  if (obs_bulk(NA, O)) warp_flush_bulk(dst, nvalid, O, sbuf);
  else warp_flush(dst, nvalid, O, sbuf);
}

inline size_t obs_stage_bytes(int NA, int O) {
  return (size_t)kSmallThreads * O * sizeof(float) * obs_nbuf(NA, O);
}

// Flush staged rows whose per-lane stride P is padded to an odd number of
// floats (conflict-free row writes for any O).  With O % 4 == 0 each 16-byte
// output chunk lies inside one row: 4 scalar shared loads, one float4 store.
SS_DEV void warp_flush_padded(float* __restrict__ dst, int nvalid, int O, int P,
                              const float* __restrict__ sbuf) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  const int n = nvalid * O;
  // row = floor(q / O4) through a float reciprocal: (q + 0.5) / O4 sits at
  // least 0.5 / O4 from an integer and q <= 32 * O, so the float product
  // (relative error < 2^-22) always truncates to the exact quotient.
  if ((O & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && ((O >> 2) & ((O >> 2) - 1)) == 0) {
    // rows of a power-of-two number of 16-byte chunks: shifts, no division
    const int sh = __ffs(O >> 2) - 1;
    for (int q = lane; q < (n >> 2); q += 32) {
      const int r = q >> sh, j = (q & ((1 << sh) - 1)) << 2;
      const float* s = sbuf + r * P + j;
      __stcs(reinterpret_cast<float4*>(dst) + q, make_float4(s[0], s[1], s[2], s[3]));
    }
  } else if ((O & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
    const int O4 = O >> 2;
    const float inv = 1.0f / (float)O4;
    for (int q = lane; q < (n >> 2); q += 32) {
      const int r = __float2int_rz(__fmul_rn(__int2float_rn(q) + 0.5f, inv)), j = (q - r * O4) << 2;
      const float* s = sbuf + r * P + j;
      __stcs(reinterpret_cast<float4*>(dst) + q, make_float4(s[0], s[1], s[2], s[3]));
    }
  } else {
    const float inv = 1.0f / (float)O;
    for (int i = lane; i < n; i += 32) {
      const int r = __float2int_rz(__fmul_rn(__int2float_rn(i) + 0.5f, inv));
      __stcs(dst + i, sbuf[r * P + (i - r * O)]);
    }
  }
  __syncwarp();
}

// decode_action's continuous branch (env.py:96-98) unless the host already
// produced final forces.
SS_DEV float decode_axis(float raw, const SsEntityDesc& d, int raw_forces) {
  return raw_forces ? raw : fmul(clip_sym(raw, d.u_range), d.u_mult);
}

// Rollout kernels: resident CTAs per SM the register budget is sized for,
// and whether step s+1's actions are loaded before step s computes.
#ifndef SS_ROLLOUT_MINB
#define SS_ROLLOUT_MINB 5   // 5 x 128 threads: <= 96 registers (tools/sweep_variants.py, SWEEP_S=10)
#endif
#ifndef SS_ROLLOUT_HALF_CTA
#define SS_ROLLOUT_HALF_CTA 1
#endif
#ifndef SS_ROLLOUT_PREFETCH
#define SS_ROLLOUT_PREFETCH 1
#endif

// Per-step pointers of a fused rollout (SsRolloutIO): the step kernels'
// SmallArgs plus, for each of n_steps steps, its actions and outputs.
struct RolloutArgs {
  SmallArgs a;
  int n_steps;
  const float2* act[SS_MAX_ROLLOUT][kSmallMaxAgents];
  float* obs[SS_MAX_ROLLOUT];
  float* rew[SS_MAX_ROLLOUT];
  uint8_t* done[SS_MAX_ROLLOUT];
  const int* guard;   // [n_steps] or nullptr
};

// Step s of a rollout runs iff its NaN words 0..s are all zero (sticky).
// Steps a rollout launch runs: up to (excluding) the first step whose scan
// (or an earlier one) found a NaN.  The scans completed before the launch
// (grid_dep_sync), so one read of the S words at entry decides it.
SS_DEV int rollout_len(const int* g, int n) {
  if (g == nullptr) return n;
  for (int s = 0; s < n; ++s)
    if (g[s]) return s;
  return n;
}

int launch_spread_rollout(World& w, RolloutArgs& r, cudaStream_t st);
int launch_transport_rollout(World& w, RolloutArgs& r, cudaStream_t st);
int launch_flocking_rollout(World& w, RolloutArgs& r, cudaStream_t st);

// Host launchers, one per translation unit (a: filled by launch_small; grid /
// shmem derived from it).  Each returns an SsStatus.
int launch_spread(World& w, SmallArgs& a, cudaStream_t st);
int launch_transport(World& w, SmallArgs& a, cudaStream_t st);
int launch_dropout(World& w, SmallArgs& a, cudaStream_t st);
int launch_catalog(World& w, SmallArgs& a, cudaStream_t st);
int launch_flocking(World& w, SmallArgs& a, cudaStream_t st);

}  // namespace ss
