// ss_transport.cu — fused Env.step of transport / reverse_transport
// (scenarios/transport.py, reverse_transport.py) and dropout (dropout.py).
#include "ss_small.cuh"

namespace ss {

// ---------------------------------------------------------------------------
// transport (scenarios/transport.py): NA agents (dyn 0..NA-1), package box
// (entity NA, dyn row NA), goal marker (entity NA+1, stat row 0).
// Pairs, lexicographic: for i: agents j>i (sphere-sphere), then (i, package)
// (sphere-box).  sc[0] = box half length (as f32 of the python double) ,
// sc[1] = half width, sc[2] = f32(success_dist); the doubles are passed via
// si-packed bits: see make_small_args.
// ---------------------------------------------------------------------------
// REV = 1: reverse_transport (catalog scenarios/reverse_transport.py): the
// same world (agents inside a hollow crate), observation
// [x, y, vx, vy, crate - self, crate vel, goal - crate] (O = 10).
// One physics (sub-)step of transport for env e: forces from `act` (decoded
// actions + gravity), contacts in the reference's pair order (agent pairs,
// then agent i vs the package box), integrate; STORE: write each state row
// as soon as it is final.
//
// Contacts in three phases, so the expensive part of collision_force (sqrt,
// two divisions, softplus) exists once in the code and runs with every lane
// of the warp busy: (1) per pair, unrolled: the cheap geometry and the
// activity test (dynamics.py:46-50), the offset of each active pair parked
// in the warp's shared scratch `scr` (float2 per pair, lane-interleaved);
// (2) each lane walks ITS active pairs (a bitmask) through one copy of the
// force code, so lanes with different active pairs share the instructions
// instead of diverging over ten inlined copies; (3) per pair, unrolled, the
// forces are summed in the reference's pair order.  Same operations on the
// same values: bitwise the one-pass result.
template <int NA>
constexpr int transport_pairs() { return NA * (NA - 1) / 2 + NA; }

template <int NA, bool STORE>
SS_DEV void transport_physics(float (&px)[NA + 1], float (&py)[NA + 1], float (&vx)[NA + 1],
                              float (&vy)[NA + 1], const float2 (&act)[NA], float ca, float sa,
                              const SmallArgs& a, int64_t B, int64_t e, float2* scr) {
  constexpr int P = transport_pairs<NA>();
  static_assert(P <= 64, "pair mask is 64 bits");
  const double hx = a.sd[0], hy = a.sd[1];
  float fx[NA + 1], fy[NA + 1];
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const SsEntityDesc& d = tmpl_ent(a, i);
    fx[i] = decode_axis(act[i].x, d, a.raw_forces);
    fy[i] = decode_axis(act[i].y, d, a.raw_forces);
  }
  fx[NA] = 0.0f; fy[NA] = 0.0f;
  if (a.ph.has_gravity) {
#pragma unroll
    for (int i = 0; i <= NA; ++i) {
      fx[i] = fadd(fx[i], tmpl_ent(a, i).grav_x); fy[i] = fadd(fy[i], tmpl_ent(a, i).grav_y);
    }
  }
  // (1) geometry + activity, pair order
  uint64_t act_mask = 0;
  {
    int p = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
#pragma unroll
      for (int j = i + 1; j < NA; ++j, ++p) {
        const float x = fsub(px[i], px[j]), y = fsub(py[i], py[j]);
        if (fadd(fmul(x, x), fmul(y, y)) <= tmpl_pair(a, p).d2_act) {
          act_mask |= 1ull << p;
          scr[p * 32] = make_float2(x, y);
        }
      }
      float qx, qy;   // agent i vs package (sphere-box): closest point on the box
      closest_point_on_box(px[i], py[i], px[NA], py[NA], ca, sa, hx, hy, qx, qy);
      const float x = fsub(px[i], qx), y = fsub(py[i], qy);
      if (fadd(fmul(x, x), fmul(y, y)) <= tmpl_pair(a, p).d2_act) {
        act_mask |= 1ull << p;
        scr[p * 32] = make_float2(x, y);
      }
      ++p;
    }
  }
  // (2) this lane's active pairs through one copy of the force code
  for (uint64_t m = act_mask; m != 0; m &= m - 1) {
    const int p = __ffsll((long long)m) - 1;
    const SsPairDesc pr = a.pairs[p];
    const float2 xy = scr[p * 32];
    const float d = fsqrt(fadd(fmul(xy.x, xy.x), fmul(xy.y, xy.y)));
    float dx, dy;
    if (d < 1e-8f) { dx = pr.sign; dy = 0.0f; }          // DEGENERATE_DIST, dynamics.py:23
    else { dx = fdiv(xy.x, d); dy = fdiv(xy.y, d); }
    const float mag = fmul(a.ph.ck, np_softplus(fdiv(fsub(pr.d_min, d), a.ph.k)));
    scr[p * 32] = make_float2(fmul(dx, mag), fmul(dy, mag));
  }
  // (3) accumulate in pair order
  {
    int p = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
#pragma unroll
      for (int j = i + 1; j <= NA; ++j, ++p) {   // j == NA: the package
        if ((act_mask >> p) & 1u) {
          const float2 c = scr[p * 32];
          fx[i] = fadd(fx[i], c.x); fy[i] = fadd(fy[i], c.y);
          fx[j] = fsub(fx[j], c.x); fy[j] = fsub(fy[j], c.y);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i <= NA; ++i) {
    const SsEntityDesc& d = tmpl_ent(a, i);
    integrate_lin(px[i], py[i], vx[i], vy[i], fx[i], fy[i], a.ph.keep, d.inv_m_dt, a.ph.dt,
                  d.max_speed);
    // single step: store each row as soon as it is final (the LSU drains
    // the stores while the next entity integrates)
    if (STORE) a.s.dyn[i * B + e] = make_float4(px[i], py[i], vx[i], vy[i]);
  }
}

// The warp's contact scratch: transport_pairs<NA>() float2 per lane inside
// the warp's own obs staging block (free until the obs rows are staged).
template <int NA, int O>
SS_DEV float2* transport_scratch(float* smem) {
  static_assert(2 * transport_pairs<NA>() <= obs_nbuf(NA, O) * O, "scratch fits the warp's staging");
  return reinterpret_cast<float2*>(obs_stage_base(smem, NA, O)) + (threadIdx.x & 31);
}

// Observation row of agent i: [x, y, vx, vy, package - self, goal - self,
// package - goal, package vel] (REV: [x, y, vx, vy, crate - self, crate vel,
// goal - crate]).
template <int NA, int REV>
SS_DEV void transport_obs_row(int i, float* row, const float (&px)[NA + 1], const float (&py)[NA + 1],
                              const float (&vx)[NA + 1], const float (&vy)[NA + 1], float gx, float gy) {
  if (REV) {
    row[0] = px[i]; row[1] = py[i]; row[2] = vx[i]; row[3] = vy[i];
    row[4] = fsub(px[NA], px[i]); row[5] = fsub(py[NA], py[i]);
    row[6] = vx[NA]; row[7] = vy[NA];
    row[8] = fsub(gx, px[NA]); row[9] = fsub(gy, py[NA]);
  } else {
    // 48-byte rows: three 16-byte shared stores (conflict-free per
    // quarter warp: lane offsets 48 l span distinct bank quads)
    float4* r4 = reinterpret_cast<float4*>(row);
    r4[0] = make_float4(px[i], py[i], vx[i], vy[i]);
    r4[1] = make_float4(fsub(px[NA], px[i]), fsub(py[NA], py[i]), fsub(gx, px[i]), fsub(gy, py[i]));
    r4[2] = make_float4(fsub(px[NA], gx), fsub(py[NA], gy), vx[NA], vy[NA]);
  }
}

template <int NA, int REV, bool MS>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_transport(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = REV ? 10 : 12;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  float px[NA + 1], py[NA + 1], vx[NA + 1], vy[NA + 1];
  float gx = 0.f, gy = 0.f, prot = 0.f;
  float2 u[NA];
  int64_t steps = 0;
  if (valid) {
    // every global load of the step issued up front
#pragma unroll
    for (int i = 0; i <= NA; ++i) {
      const float4 q = a.s.dyn[i * B + e];
      px[i] = q.x; py[i] = q.y; vx[i] = q.z; vy[i] = q.w;
    }
    const float2 g = a.s.stat[e];
    gx = g.x; gy = g.y;
    if (a.mode & SS_DO_PHYSICS) {
      prot = a.s.rot[NA * B + e].x;
#pragma unroll
      for (int i = 0; i < NA; ++i) u[i] = a.act[i][e];
    }
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_PHYSICS)) {
    float ca, sa;
    if (prot == 0.0f) { ca = 1.0f; sa = prot; } else { ca = np_cosf(prot); sa = np_sinf(prot); }
    float2* scr = transport_scratch<NA, O>(smem);
    transport_physics<NA, !MS>(px, py, vx, vy, u, ca, sa, a, B, e, scr);
    // further physics sub-steps (PhysK.substeps > 1: the MS instantiation,
    // so the reference's single step keeps its register budget) reload the
    // held actions instead of keeping them live across the first one
    if (MS) for (int sub = 1; sub < a.ph.substeps; ++sub) {
      float2 ur[NA];
#pragma unroll
      for (int i = 0; i < NA; ++i) ur[i] = a.act[i][e];
      transport_physics<NA, false>(px, py, vx, vy, ur, ca, sa, a, B, e, scr);
    }
    if (MS) {
#pragma unroll
      for (int i = 0; i <= NA; ++i) a.s.dyn[i * B + e] = make_float4(px[i], py[i], vx[i], vy[i]);
    }
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  if (valid && (a.mode & (SS_DO_REWARD | SS_DO_DONE))) {
    const float gap = norm2(fsub(px[NA], gx), fsub(py[NA], gy));
    if (a.mode & SS_DO_REWARD) {
#pragma unroll
      for (int i = 0; i < NA; ++i) __stcs(a.rew + i * B + e, -gap);
    }
    if (a.mode & SS_DO_DONE) a.done[e] = (uint8_t)((gap < a.sc[2]) | (steps >= a.ph.max_steps));
  }
  if (a.mode & SS_DO_OBS) {
    float* sbuf = nullptr;
    float* row = nullptr;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
    __syncwarp();   // every lane is done with its contact scratch in the staging
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      sbuf = obs_stage(smem, i, NA, O);
      row = sbuf + (threadIdx.x & 31) * O;
      if (valid) transport_obs_row<NA, REV>(i, row, px, py, vx, vy, gx, gy);
      if (nvalid > 0) obs_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, NA, O, sbuf);
    }
    obs_bulk_drain();
  }
}

// transport, fused open-loop rollout (SsRolloutIO): n_steps steps with the
// agents and the package in registers between them (the goal and the
// package's fixed rotation read once); state read once, written once.
// MINB: resident CTAs per SM the register budget targets — SS_ROLLOUT_MINB
// (96 registers) in general, 6 (80 registers) when that puts the whole grid
// in ONE wave and SS_ROLLOUT_MINB would not (100k envs: 782 CTAs vs 740 /
// 888 slots; 8.9 -> 8.2 us per step; at 1M the 96-register build is faster).
template <int NA, int REV, int MINB>
__global__ void __launch_bounds__(kSmallThreads, MINB) k_transport_rollout(const RolloutArgs r) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  const SmallArgs& a = r.a;
  constexpr int O = REV ? 10 : 12;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  const int64_t e0 = e - (threadIdx.x & 31);
  const int nvalid = (int)min((int64_t)32, B - e0);
  float px[NA + 1], py[NA + 1], vx[NA + 1], vy[NA + 1];
  float gx = 0.f, gy = 0.f, prot = 0.f;
  int64_t steps = 0;
  if (valid) {
#pragma unroll
    for (int i = 0; i <= NA; ++i) {
      const float4 q = a.s.dyn[i * B + e];
      px[i] = q.x; py[i] = q.y; vx[i] = q.z; vy[i] = q.w;
    }
    const float2 g = a.s.stat[e];
    gx = g.x; gy = g.y;
    prot = a.s.rot[NA * B + e].x;
    steps = a.s.step_count[e];
  }
  float ca, sa;
  if (prot == 0.0f) { ca = 1.0f; sa = prot; } else { ca = np_cosf(prot); sa = np_sinf(prot); }
  const int n_run = rollout_len(r.guard, r.n_steps);   // uniform over the grid
  float2 u[NA];
  if (valid && n_run > 0) {
#pragma unroll
    for (int i = 0; i < NA; ++i) u[i] = __ldcs(r.act[0][i] + e);
  }
  for (int s = 0; s < n_run; ++s) {
    float2 un[NA];   // the next step's actions, in flight during this step
    if (SS_ROLLOUT_PREFETCH && valid && s + 1 < n_run) {
#pragma unroll
      for (int i = 0; i < NA; ++i) un[i] = __ldcs(r.act[s + 1][i] + e);
    }
    if (s > 0) {   // the previous step's bulk stores must have read the staging
      obs_bulk_drain();
      __syncwarp();
    }
    if (valid) {
      transport_physics<NA, false>(px, py, vx, vy, u, ca, sa, a, B, e, transport_scratch<NA, O>(smem));
      steps += 1;
      const float gap = norm2(fsub(px[NA], gx), fsub(py[NA], gy));
#pragma unroll
      for (int i = 0; i < NA; ++i) __stcs(r.rew[s] + i * B + e, -gap);
      r.done[s][e] = (uint8_t)((gap < a.sc[2]) | (steps >= a.ph.max_steps));
    }
    __syncwarp();   // every lane is done with its contact scratch in the staging
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      float* sbuf = obs_stage(smem, i, NA, O);
      float* row = sbuf + (threadIdx.x & 31) * O;
      if (valid) transport_obs_row<NA, REV>(i, row, px, py, vx, vy, gx, gy);
      if (nvalid > 0) obs_flush(r.obs[s] + i * a.obs_stride + e0 * O, nvalid, NA, O, sbuf);
    }
    if (SS_ROLLOUT_PREFETCH) {
#pragma unroll
      for (int i = 0; i < NA; ++i) u[i] = un[i];
    } else if (valid && s + 1 < n_run) {
#pragma unroll
      for (int i = 0; i < NA; ++i) u[i] = __ldcs(r.act[s + 1][i] + e);
    }
  }
  if (valid) {
#pragma unroll
    for (int i = 0; i <= NA; ++i) a.s.dyn[i * B + e] = make_float4(px[i], py[i], vx[i], vy[i]);
    a.s.step_count[e] = steps;
  }
  obs_bulk_drain();
}

// ---------------------------------------------------------------------------
// dropout (catalog scenarios/dropout.py): NA non-collidable agents (dyn
// 0..NA-1), goal marker (stat row 0); no pairs.  Reward (shared):
// float64(any agent within reach) - energy_coeff * spent, spent = the float64
// sum over agents, in order, of fx*fx then fy*fy (float32 squares of the
// decoded actions, promoted); done = reached.  spent is kept in flag words 0
// and 1 (double bits) so a reward-only launch sees the last step's value.
// sc[3] = squared bound of f32(reach); sd[0] = energy_coeff.
// Observation: [x, y, vx, vy, goal - self, (other - self)].
// ---------------------------------------------------------------------------
template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_dropout(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 4 + 2 * NA;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  float px[NA], py[NA], vx[NA], vy[NA];
  float2 u[NA];
  float gx = 0.f, gy = 0.f;
  int64_t steps = 0;
  uint32_t lo = 0u, hi = 0u;
  if (valid) {
    // every global load of the step issued up front
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const float4 q = a.s.dyn[i * B + e];
      px[i] = q.x; py[i] = q.y; vx[i] = q.z; vy[i] = q.w;
    }
    const float2 g = a.s.stat[e];
    gx = g.x; gy = g.y;
    if (a.mode & SS_DO_PHYSICS) {
#pragma unroll
      for (int i = 0; i < NA; ++i) u[i] = a.act[i][e];
    } else if (a.mode & SS_DO_REWARD) {
      lo = a.s.flags[e];
      hi = a.s.flags[B + e];
    }
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  double spent = __hiloint2double((int)hi, (int)lo);
  if (valid && (a.mode & SS_DO_PHYSICS)) {
    spent = 0.0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const SsEntityDesc& d = a.ents[i];
      float fx = decode_axis(u[i].x, d, a.raw_forces), fy = decode_axis(u[i].y, d, a.raw_forces);
      spent = dadd_rn(dadd_rn(spent, (double)fmul(fx, fx)), (double)fmul(fy, fy));
      if (a.ph.has_gravity) { fx = fadd(fx, d.grav_x); fy = fadd(fy, d.grav_y); }
      for (int sub = 0; sub < a.ph.substeps; ++sub)   // no pairs: sub-steps are independent
        integrate_lin(px[i], py[i], vx[i], vy[i], fx, fy, a.ph.keep, d.inv_m_dt, a.ph.dt, d.max_speed);
      a.s.dyn[i * B + e] = make_float4(px[i], py[i], vx[i], vy[i]);
    }
    a.s.flags[e] = (uint32_t)__double2loint(spent);
    a.s.flags[B + e] = (uint32_t)__double2hiint(spent);
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  bool reached = false;
  if (valid) {
#pragma unroll
    for (int i = 0; i < NA; ++i) reached |= sqnorm(fsub(px[i], gx), fsub(py[i], gy)) <= a.sc[3];
  }
  if (valid && (a.mode & SS_DO_REWARD)) {
    const float r = (float)dsub_rn(reached ? 1.0 : 0.0, dmul_rn(a.sd[0], spent));
#pragma unroll
    for (int i = 0; i < NA; ++i) __stcs(a.rew + i * B + e, r);
  }
  if (valid && (a.mode & SS_DO_DONE)) a.done[e] = (uint8_t)(reached | (steps >= a.ph.max_steps));
  if (a.mode & SS_DO_OBS) {
    float* sbuf = nullptr;
    float* row = nullptr;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      sbuf = obs_stage(smem, i, NA, O);
      row = sbuf + (threadIdx.x & 31) * O;
      if (valid) {
        row[0] = px[i]; row[1] = py[i]; row[2] = vx[i]; row[3] = vy[i];
        row[4] = fsub(gx, px[i]); row[5] = fsub(gy, py[i]);
        int c = 6;
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          if (o == i) continue;
          row[c++] = fsub(px[o], px[i]); row[c++] = fsub(py[o], py[i]);
        }
      }
      if (nvalid > 0) obs_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, NA, O, sbuf);
    }
    obs_bulk_drain();
  }
}

int launch_transport(World& w, SmallArgs& a, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const bool ms = a.ph.substeps > 1;
  const unsigned grid = (unsigned)((w.d.batch + kSmallThreads - 1) / kSmallThreads);
  const size_t shmem = obs_stage_bytes(w.d.n_agents, w.d.obs_dim);
#define SS_CASE(n)                                                                                   \
  case n:                                                                                            \
    if (ms) {                                                                                        \
      if (w.d.si[1]) launch_step(k_transport<n, 1, true>, dim3(grid), dim3(kSmallThreads), shmem, st, a); \
      else launch_step(k_transport<n, 0, true>, dim3(grid), dim3(kSmallThreads), shmem, st, a);           \
    } else {                                                                                         \
      if (w.d.si[1]) launch_step(k_transport<n, 1, false>, dim3(grid), dim3(kSmallThreads), shmem, st, a); \
      else launch_step(k_transport<n, 0, false>, dim3(grid), dim3(kSmallThreads), shmem, st, a);           \
    }                                                                                                \
    break;
  switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
  return cuda_status(cudaGetLastError(), "transport step launch");
}

int launch_transport_rollout(World& w, RolloutArgs& r, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const unsigned grid = (unsigned)((w.d.batch + kSmallThreads - 1) / kSmallThreads);
  const size_t shmem = obs_stage_bytes(NA, w.d.obs_dim);
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const bool one_wave6 = grid <= (unsigned)(6 * sms) && grid > (unsigned)(SS_ROLLOUT_MINB * sms);
  // one-wave case: SS_ROLLOUT_HALF_CTA splits the grid into 64-thread CTAs
  // (same registers and shared memory per thread), so the SMs get 10-11
  // CTAs each instead of 5-6 (less tail imbalance inside the single wave)
  const unsigned bt = (one_wave6 && SS_ROLLOUT_HALF_CTA) ? kSmallThreads / 2 : kSmallThreads;
  const unsigned g1 = (unsigned)((w.d.batch + bt - 1) / bt);
  const size_t sh1 = shmem * bt / kSmallThreads;
#define SS_CASE(n)                                                                                   \
  case n:                                                                                            \
    if (one_wave6) {                                                                                       \
      if (w.d.si[1]) launch_step(k_transport_rollout<n, 1, 6>, dim3(g1), dim3(bt), sh1, st, r);             \
      else launch_step(k_transport_rollout<n, 0, 6>, dim3(g1), dim3(bt), sh1, st, r);                       \
    } else if (w.d.si[1]) {                                                                                \
      launch_step(k_transport_rollout<n, 1, SS_ROLLOUT_MINB>, dim3(grid), dim3(kSmallThreads), shmem, st, r); \
    } else {                                                                                               \
      launch_step(k_transport_rollout<n, 0, SS_ROLLOUT_MINB>, dim3(grid), dim3(kSmallThreads), shmem, st, r); \
    }                                                                                                      \
    break;
  switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
  return cuda_status(cudaGetLastError(), "transport rollout launch");
}

int launch_dropout(World& w, SmallArgs& a, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const unsigned grid = (unsigned)((w.d.batch + kSmallThreads - 1) / kSmallThreads);
  const size_t shmem = obs_stage_bytes(w.d.n_agents, w.d.obs_dim);
#define SS_CASE(n) case n: launch_step(k_dropout<n>, dim3(grid), dim3(kSmallThreads), shmem, st, a); break;
  switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
  return cuda_status(cudaGetLastError(), "dropout step launch");
}

}  // namespace ss
