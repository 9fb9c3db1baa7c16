// ss_catalog.cu — fused Env.step of the line / box catalog tasks (wheel,
// give_way, passage, balance, waterfall, football): world_step (the shared
// env_physics of ss_physics.cuh, sub-steps included) and the task's count,
// reward, done and observation in one launch; football's scripted reds in-kernel.
#include "ss_physics.cuh"
#include "ss_small.cuh"

namespace ss {

// world_step (dynamics.py:123-184) for one env of a line / box catalog task,
// inside its fused kernel (ss_physics.cuh env_physics: any pair list,
// torques, gravity, sub-steps).  Agent i's force is decode_action of its raw
// action (or the host-decoded force); the last n_script agents, when their
// action_script runs in the kernel (!raw_forces), take script[i - first]
// instead.  Accumulators after the obs staging.  One out-of-line copy for
// every catalog kernel (the generic closest-point code is large).
constexpr int kMaxKernelScripts = 4;
struct ScriptForces { float2 f[kMaxKernelScripts]; };

__device__ __noinline__ void catalog_physics(const SmallArgs& a, int NA, int n_script, int64_t e,
                                             float* smem_base, const ScriptForces sf) {
  float* acc = smem_base + a.acc_off;
  const int first = NA - n_script;
  env_physics(a.s, a.ph, a.ents, a.pairs, a.E, a.P, nullptr, 0, NA, e, acc, kSmallThreads, threadIdx.x,
              [&](int i, float& fx, float& fy) {
    if (i >= first && !a.raw_forces) {
      const float2 f = sf.f[i - first];
      fx = f.x; fy = f.y;
      return true;
    }
    if (a.act[i] == nullptr) return false;
    const float2 u = a.act[i][e];
    fx = decode_axis(u.x, a.ents[i], a.raw_forces);
    fy = decode_axis(u.y, a.ents[i], a.raw_forces);
    return true;
  });
}

// ---------------------------------------------------------------------------
// wheel (catalog scenarios/wheel.py): NA agents (dyn 0..NA-1) and a pinned
// rotatable rod (entity NA, stat row 0).  Physics (sphere-line contacts and
// the rod's torque) is world_step's (k_generic_physics, launched first);
// this kernel does the rest of the step: count, reward -|w - target| (float32,
// shared), horizon done, observation
// [x, y, vx, vy, rod - self, cos(rot), sin(rot), w, target] with numpy's
// float32 cos/sin.  sc[0] = f32(target_spin).
// ---------------------------------------------------------------------------
template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_wheel(const __grid_constant__ SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 10;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  if (valid && (a.mode & SS_DO_PHYSICS)) catalog_physics(a, NA, 0, e, smem, ScriptForces());
  int64_t steps = 0;
  float2 rod = make_float2(0.f, 0.f), rw = rod;
  if (valid) {
    rod = a.s.stat[e];
    rw = a.s.rot[NA * B + e];
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  if (valid && (a.mode & SS_DO_REWARD)) {
    const float r = -fabsf(fsub(rw.y, a.sc[0]));
#pragma unroll
    for (int i = 0; i < NA; ++i) __stcs(a.rew + i * B + e, r);
  }
  if (valid && (a.mode & SS_DO_DONE)) a.done[e] = (uint8_t)(steps >= a.ph.max_steps);
  if (a.mode & SS_DO_OBS) {
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
    const float c = valid ? np_cosf(rw.x) : 0.f, sn = valid ? np_sinf(rw.x) : 0.f;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) {
        const float4 q = a.s.dyn[i * B + e];
        row[0] = q.x; row[1] = q.y; row[2] = q.z; row[3] = q.w;
        row[4] = fsub(rod.x, q.x); row[5] = fsub(rod.y, q.y);
        row[6] = c; row[7] = sn; row[8] = rw.y; row[9] = a.sc[0];
      }
      if (nvalid > 0) warp_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
}

// ---------------------------------------------------------------------------
// give_way (catalog scenarios/give_way.py): agents 0, 1 (dyn rows 0, 1),
// goals 0, 1 (stat rows 0, 1), six walls.  Physics (sphere-line contacts) is
// world_step's; this kernel: count, reward for agent k
// f32(-float64(gap_k) + 5.0 * float64(gap_k < f32(0.15))), done = both gaps
// < f32(0.15), observation [x, y, vx, vy, goal_k - self, other - self, other
// vel, f32(alcove_x - float64(x)), f32(alcove_y - float64(y))].
// sc[0] = f32(0.15); sd[0], sd[1] = alcove (python doubles).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_give_way(const __grid_constant__ SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 12;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  if (valid && (a.mode & SS_DO_PHYSICS)) catalog_physics(a, 2, 0, e, smem, ScriptForces());
  float4 ag[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
  float2 goal[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  int64_t steps = 0;
  if (valid) {
    ag[0] = a.s.dyn[e]; ag[1] = a.s.dyn[B + e];
    goal[0] = a.s.stat[e]; goal[1] = a.s.stat[B + e];
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  const float thr = a.sc[0];
  float gap[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) gap[k] = norm2(fsub(ag[k].x, goal[k].x), fsub(ag[k].y, goal[k].y));
  if (valid && (a.mode & SS_DO_REWARD)) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      __stcs(a.rew + k * B + e, (float)dadd_rn(-(double)gap[k], gap[k] < thr ? 5.0 : 0.0));
  }
  if (valid && (a.mode & SS_DO_DONE))
    a.done[e] = (uint8_t)(((gap[0] < thr) & (gap[1] < thr)) | (steps >= a.ph.max_steps));
  if (a.mode & SS_DO_OBS) {
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (valid) {
        const float4 me = ag[k], ot = ag[1 - k];
        row[0] = me.x; row[1] = me.y; row[2] = me.z; row[3] = me.w;
        row[4] = fsub(goal[k].x, me.x); row[5] = fsub(goal[k].y, me.y);
        row[6] = fsub(ot.x, me.x); row[7] = fsub(ot.y, me.y);
        row[8] = ot.z; row[9] = ot.w;
        row[10] = (float)dsub_rn(a.sd[0], (double)me.x);
        row[11] = (float)dsub_rn(a.sd[1], (double)me.y);
      }
      if (nvalid > 0) warp_flush(a.obs + k * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
}

// ---------------------------------------------------------------------------
// passage (catalog scenarios/passage.py): NA agents (dyn 0..NA-1), their
// slots (stat rows 0..NA-1), three wall segments.  Physics is world_step's;
// this kernel: count, reward -gap_k - f32(pen) * #touching teammates
// (float32), done = every agent within f32(0.05) of its slot, observation
// [x, y, vx, vy, slot - self, (f32(gap_x - float64(x)), 0 - y) per wall gap,
// (other - self)].  sc[0] = f32 touch distance, sc[1] = f32(pen),
// sc[2] = f32(0.05); sd[0], sd[1] = gap centres (python doubles).
// ---------------------------------------------------------------------------
template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_passage(const __grid_constant__ SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 10 + 2 * (NA - 1);
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  if (valid && (a.mode & SS_DO_PHYSICS)) catalog_physics(a, NA, 0, e, smem, ScriptForces());
  float4 ag[NA];
  float2 slot[NA];
  int64_t steps = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) { ag[i] = make_float4(0.f, 0.f, 0.f, 0.f); slot[i] = make_float2(0.f, 0.f); }
  if (valid) {
#pragma unroll
    for (int i = 0; i < NA; ++i) { ag[i] = a.s.dyn[i * B + e]; slot[i] = a.s.stat[i * B + e]; }
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  float gap[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) gap[i] = norm2(fsub(ag[i].x, slot[i].x), fsub(ag[i].y, slot[i].y));
  if (valid && (a.mode & SS_DO_REWARD)) {
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      float cnt = 0.0f;   // common.contact_count: float32 sum in agent order
#pragma unroll
      for (int o = 0; o < NA; ++o) {
        if (o == i) continue;
        cnt = fadd(cnt, norm2(fsub(ag[i].x, ag[o].x), fsub(ag[i].y, ag[o].y)) <= a.sc[0] ? 1.0f : 0.0f);
      }
      __stcs(a.rew + i * B + e, fsub(-gap[i], fmul(a.sc[1], cnt)));
    }
  }
  if (valid && (a.mode & SS_DO_DONE)) {
    bool all = true;
#pragma unroll
    for (int i = 0; i < NA; ++i) all &= gap[i] < a.sc[2];
    a.done[e] = (uint8_t)(all | (steps >= a.ph.max_steps));
  }
  if (a.mode & SS_DO_OBS) {
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) {
        const float4 me = ag[i];
        row[0] = me.x; row[1] = me.y; row[2] = me.z; row[3] = me.w;
        row[4] = fsub(slot[i].x, me.x); row[5] = fsub(slot[i].y, me.y);
        row[6] = (float)dsub_rn(a.sd[0], (double)me.x); row[7] = fsub(0.0f, me.y);
        row[8] = (float)dsub_rn(a.sd[1], (double)me.x); row[9] = fsub(0.0f, me.y);
        int c = 10;
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          if (o == i) continue;
          row[c++] = fsub(ag[o].x, me.x); row[c++] = fsub(ag[o].y, me.y);
        }
      }
      if (nvalid > 0) warp_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
}

// ---------------------------------------------------------------------------
// balance (catalog scenarios/balance.py): NA agents (dyn 0..NA-1), tray
// (entity NA, dyn row NA, rotatable), ball (dyn row NA+1), goal (stat row 0),
// floor.  Physics (gravity, sphere-line contacts, the tray's torque) is
// world_step's; this kernel: count, reward f32(-float64(gap) - 5 *
// float64(ball.y < f32(floor + r + 0.02))) with gap = |ball - goal|, done =
// gap < f32(0.08), observation [x, y, vx, vy, tray - self, cos, sin (numpy
// float32), tray w, tray vel, ball - self, ball vel, goal - ball].
// sc[0] = f32 drop height, sc[1] = f32(0.08).
// ---------------------------------------------------------------------------
template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_balance(const __grid_constant__ SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 17;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  if (valid && (a.mode & SS_DO_PHYSICS)) catalog_physics(a, NA, 0, e, smem, ScriptForces());
  float4 tray = make_float4(0.f, 0.f, 0.f, 0.f), ball = tray;
  float2 trw = make_float2(0.f, 0.f), goal = trw;
  int64_t steps = 0;
  if (valid) {
    tray = a.s.dyn[NA * B + e];
    ball = a.s.dyn[(NA + 1) * B + e];
    trw = a.s.rot[NA * B + e];
    goal = a.s.stat[e];
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  const float gap = norm2(fsub(ball.x, goal.x), fsub(ball.y, goal.y));
  if (valid && (a.mode & SS_DO_REWARD)) {
    const float r = (float)dsub_rn(-(double)gap, ball.y < a.sc[0] ? 5.0 : 0.0);
#pragma unroll
    for (int i = 0; i < NA; ++i) __stcs(a.rew + i * B + e, r);
  }
  if (valid && (a.mode & SS_DO_DONE)) a.done[e] = (uint8_t)((gap < a.sc[1]) | (steps >= a.ph.max_steps));
  if (a.mode & SS_DO_OBS) {
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
    const float c = valid ? np_cosf(trw.x) : 0.f, sn = valid ? np_sinf(trw.x) : 0.f;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) {
        const float4 q = a.s.dyn[i * B + e];
        row[0] = q.x; row[1] = q.y; row[2] = q.z; row[3] = q.w;
        row[4] = fsub(tray.x, q.x); row[5] = fsub(tray.y, q.y);
        row[6] = c; row[7] = sn; row[8] = trw.y; row[9] = tray.z; row[10] = tray.w;
        row[11] = fsub(ball.x, q.x); row[12] = fsub(ball.y, q.y);
        row[13] = ball.z; row[14] = ball.w;
        row[15] = fsub(goal.x, ball.x); row[16] = fsub(goal.y, ball.y);
      }
      if (nvalid > 0) warp_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
}

// ---------------------------------------------------------------------------
// waterfall (catalog scenarios/waterfall.py): NA agents (dyn 0..NA-1), basin
// (stat row 0), NB box baffles (entities NA+1.., stat rows 1..NB).  Physics
// (gravity, sphere-box contacts) is world_step's; this kernel: count, reward
// f32(-float64(gap) - pen * (float64(#touching teammates) + float64 sum of
// block bumps)), a bump = |self - closest point on the block| <= f32(r);
// done = every agent within f32(0.2) of the basin; observation [x, y, vx, vy,
// basin - self, (block_k - self)].  sc[0] = f32 touch distance, sc[1] =
// f32(agent radius), sc[2] = f32(0.2); sd[0] = pen (python double); si[2] = NB.
// ---------------------------------------------------------------------------
constexpr int kWaterfallMaxBlocks = 8;

template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_waterfall(const __grid_constant__ SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  const int NB = a.si[2];
  const int O = a.obs_dim;   // 6 + 2 NB
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  if (valid && (a.mode & SS_DO_PHYSICS)) catalog_physics(a, NA, 0, e, smem, ScriptForces());
  float4 ag[NA];
  float2 basin = make_float2(0.f, 0.f);
  float2 blk[kWaterfallMaxBlocks];
  int64_t steps = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) ag[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kWaterfallMaxBlocks; ++k) blk[k] = make_float2(0.f, 0.f);
  if (valid) {
#pragma unroll
    for (int i = 0; i < NA; ++i) ag[i] = a.s.dyn[i * B + e];
    basin = a.s.stat[e];
#pragma unroll
    for (int k = 0; k < kWaterfallMaxBlocks; ++k)
      if (k < NB) blk[k] = a.s.stat[(1 + k) * B + e];
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  float gap[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) gap[i] = norm2(fsub(ag[i].x, basin.x), fsub(ag[i].y, basin.y));
  if (valid && (a.mode & SS_DO_REWARD)) {
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      float cnt = 0.0f;   // common.contact_count: float32 sum in agent order
#pragma unroll
      for (int o = 0; o < NA; ++o) {
        if (o == i) continue;
        cnt = fadd(cnt, norm2(fsub(ag[i].x, ag[o].x), fsub(ag[i].y, ag[o].y)) <= a.sc[0] ? 1.0f : 0.0f);
      }
      double bumps = 0.0;  // _block_bumps: float64 count in block order
      const SsEntityDesc& da = a.ents[i];
      ShapeK sa;
      sa.kind = da.shape; sa.d0 = da.dim0; sa.d1 = da.dim1;
      const V2 pa = v2(ag[i].x, ag[i].y);
      const float ra = a.s.rot[i * B + e].x;
      for (int k = 0; k < NB; ++k) {
        const SsEntityDesc& db = a.ents[NA + 1 + k];
        ShapeK sb;
        sb.kind = db.shape; sb.d0 = db.dim0; sb.d1 = db.dim1;
        V2 oa, ob;
        closest_points(pa, ra, sa, v2(blk[k].x, blk[k].y), a.s.rot[(NA + 1 + k) * B + e].x, sb, oa, ob);
        bumps = dadd_rn(bumps, norm2(fsub(pa.x, ob.x), fsub(pa.y, ob.y)) <= a.sc[1] ? 1.0 : 0.0);
      }
      const double b = dadd_rn((double)cnt, bumps);
      __stcs(a.rew + i * B + e, (float)dsub_rn(-(double)gap[i], dmul_rn(a.sd[0], b)));
    }
  }
  if (valid && (a.mode & SS_DO_DONE)) {
    bool all = true;
#pragma unroll
    for (int i = 0; i < NA; ++i) all &= gap[i] < a.sc[2];
    a.done[e] = (uint8_t)(all | (steps >= a.ph.max_steps));
  }
  if (a.mode & SS_DO_OBS) {
    const int P = O | 1;
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * P);
    float* row = sbuf + (threadIdx.x & 31) * P;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) {
        const float4 me = ag[i];
        row[0] = me.x; row[1] = me.y; row[2] = me.z; row[3] = me.w;
        row[4] = fsub(basin.x, me.x); row[5] = fsub(basin.y, me.y);
#pragma unroll
        for (int k = 0; k < kWaterfallMaxBlocks; ++k)
          if (k < NB) { row[6 + 2 * k] = fsub(blk[k].x, me.x); row[7 + 2 * k] = fsub(blk[k].y, me.y); }
      }
      if (nvalid > 0) warp_flush_padded(a.obs + i * a.obs_stride + e0 * O, nvalid, O, P, sbuf);
    }
  }
}

// ---------------------------------------------------------------------------
// football (catalog scenarios/football.py): NA = 2 NT agents — blues
// 0..NT-1 (controlled), reds NT..NA-1 (scripted: their forces come from the
// host script, decoded before world_step) — ball (dyn row NA), 12 walls.
// Physics is world_step's; this kernel: count, reward for blues
// f32(10 * right - 10 * left - float64(f32(0.1) * |ball - (hx, 0)|)), 0 for
// reds, done = right | left (ball beyond -/+ f32(hx + 0.04)), observation
// [x, y, vx, vy, ball - self, ball vel, (mate - self), (foe - self),
// f32(attack_x - float64(x)), 0 - y].  sc[0] = f32(hx + 0.04), sc[1] =
// f32(0.1), sc[2] = f32(hx); sd[0] = hx (python double).
// ---------------------------------------------------------------------------
template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_football(const __grid_constant__ SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int NT = NA / 2;
  constexpr int O = 4 + 2 + 2 + 2 * (NA - 1) + 2;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  if (valid && (a.mode & SS_DO_PHYSICS)) {
    // the reds' chase script (football.py:31-47) on the pre-step state, run
    // here unless the host already decoded every agent (raw_forces): the
    // nearer red (first minimum of |red - ball|) aims 0.08 behind the ball,
    // the other holds the post (-0.75, 0); 3 * aim clipped to +-u_range,
    // times u_multiplier, all float32
    ScriptForces sf;
    if (!a.raw_forces) {
      const float4 bl = a.s.dyn[NA * B + e];
      float2 rp[NT];
      float dist[NT];
#pragma unroll
      for (int r = 0; r < NT; ++r) {
        const float4 q = a.s.dyn[(NT + r) * B + e];
        rp[r] = make_float2(q.x, q.y);
        dist[r] = norm2(fsub(q.x, bl.x), fsub(q.y, bl.y));
      }
      int best = 0;
#pragma unroll
      for (int r = 1; r < NT; ++r) if (dist[r] < dist[best]) best = r;
#pragma unroll
      for (int r = 0; r < NT; ++r) {
        const bool closer = best == r;
        const float tx = closer ? fsub(fadd(bl.x, 0.08f), rp[r].x) : fsub(-0.75f, rp[r].x);
        const float ty = closer ? fsub(fadd(bl.y, 0.0f), rp[r].y) : fsub(0.0f, rp[r].y);
        const SsEntityDesc& d = a.ents[NT + r];
        sf.f[r] = make_float2(fmul(clip_sym(fmul(3.0f, tx), d.u_range), d.u_mult),
                              fmul(clip_sym(fmul(3.0f, ty), d.u_range), d.u_mult));
      }
    }
    catalog_physics(a, NA, NT, e, smem, sf);
  }
  float4 ag[NA], ball = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t steps = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) ag[i] = ball;
  if (valid) {
#pragma unroll
    for (int i = 0; i < NA; ++i) ag[i] = a.s.dyn[i * B + e];
    ball = a.s.dyn[NA * B + e];
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  const bool right = ball.x > a.sc[0], left = ball.x < -a.sc[0];
  if (valid && (a.mode & SS_DO_REWARD)) {
    const float gap = norm2(fsub(ball.x, a.sc[2]), fsub(ball.y, 0.0f));
    const double r = dsub_rn(dsub_rn(right ? 10.0 : 0.0, left ? 10.0 : 0.0), (double)fmul(a.sc[1], gap));
#pragma unroll
    for (int i = 0; i < NA; ++i) __stcs(a.rew + i * B + e, i < NT ? (float)r : 0.0f);
  }
  if (valid && (a.mode & SS_DO_DONE)) a.done[e] = (uint8_t)((right | left) | (steps >= a.ph.max_steps));
  if (a.mode & SS_DO_OBS) {
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) {
        const float4 me = ag[i];
        const bool blue = i < NT;
        row[0] = me.x; row[1] = me.y; row[2] = me.z; row[3] = me.w;
        row[4] = fsub(ball.x, me.x); row[5] = fsub(ball.y, me.y);
        row[6] = ball.z; row[7] = ball.w;
        int c = 8;
#pragma unroll
        for (int o = 0; o < NA; ++o) {          // mates, world order
          if (o == i || (o < NT) != blue) continue;
          row[c++] = fsub(ag[o].x, me.x); row[c++] = fsub(ag[o].y, me.y);
        }
#pragma unroll
        for (int o = 0; o < NA; ++o) {          // foes, world order
          if ((o < NT) == blue) continue;
          row[c++] = fsub(ag[o].x, me.x); row[c++] = fsub(ag[o].y, me.y);
        }
        row[c] = (float)dsub_rn(blue ? a.sd[0] : -a.sd[0], (double)me.x);
        row[c + 1] = fsub(0.0f, me.y);
      }
      if (nvalid > 0) warp_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
}

int launch_catalog(World& w, SmallArgs& a, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const unsigned grid = (unsigned)((w.d.batch + kSmallThreads - 1) / kSmallThreads);
  // in-launch world_step: force accumulators after the (odd-padded)
  // observation staging
  a.acc_off = kSmallThreads * (w.d.obs_dim | 1);
  const size_t cshm = (a.mode & SS_DO_PHYSICS)
      ? (size_t)(a.acc_off + 3 * a.E * kSmallThreads) * sizeof(float)
      : (size_t)kSmallThreads * (w.d.obs_dim | 1) * sizeof(float);
  if (cshm > 200 * 1024) { set_error("world too large for the fused catalog kernel"); return SS_ERR_UNSUPPORTED; }
  auto catalog_launch = [&](auto kernel) {
    if (cshm > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cshm);
    launch_step(kernel, dim3(grid), dim3(kSmallThreads), cshm, st, a);
  };
  switch (w.d.scenario) {
    case SS_SCN_WHEEL: {
#define SS_CASE(n) case n: catalog_launch(k_wheel<n>); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_GIVE_WAY: {
      if (NA != 2) {
        set_error("give_way: 2 agents");
        return SS_ERR_CONTRACT;
      }
      catalog_launch(k_give_way);
      break;
    }
    case SS_SCN_PASSAGE: {
#define SS_CASE(n) case n: catalog_launch(k_passage<n>); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_BALANCE: {
#define SS_CASE(n) case n: catalog_launch(k_balance<n>); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_WATERFALL: {
      if (w.d.si[2] > kWaterfallMaxBlocks) {
        set_error("waterfall: at most 8 blocks");
        return SS_ERR_CONTRACT;
      }
#define SS_CASE(n) case n: catalog_launch(k_waterfall<n>); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_FOOTBALL: {
      if (NA & 1) {
        set_error("football: two equal teams");
        return SS_ERR_CONTRACT;
      }
#define SS_CASE(n) case n: catalog_launch(k_football<n>); break;
      switch (NA) { SS_CASE(2) SS_CASE(4) SS_CASE(6) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    default:
      set_error("launch_catalog: not a catalog scenario");
      return SS_ERR_SCENARIO;
  }
  return cuda_status(cudaGetLastError(), "catalog step launch");
}

}  // namespace ss
