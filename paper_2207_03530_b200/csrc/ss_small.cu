// ss_small.cu — fused Env.step for the small built-in scenarios
// (simple_spread, transport, flocking): one thread per environment, the whole
// entity state of an env lives in registers for the duration of the step.
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
#include <cstdlib>

#include "ss_bulk.cuh"
#include "ss_geometry.cuh"   // (includes ss_internal.cuh)

namespace ss {

constexpr int kSmallMaxAgents = 8;
constexpr int kFlockMaxRocks = 6;
constexpr int kSmallThreads = 128;
// minimum resident CTAs per SM requested from ptxas (register budget)
#ifndef SS_SMALL_MINB
#define SS_SMALL_MINB 6   // 6 x 128 threads: <= 80 registers, best measured (tools/sweep_variants.py)
#endif

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
};

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
  if ((O & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
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

// fp64 ray vs circle (sensors.py:43-54); inf on miss.
SS_DEV double ray_circle(double ox, double oy, double dx, double dy, double cx, double cy,
                         double r2) {
  const double fx = dsub_rn(ox, cx), fy = dsub_rn(oy, cy);
  const double b = dadd_rn(dmul_rn(fx, dx), dmul_rn(fy, dy));
  const double c = dsub_rn(dadd_rn(dmul_rn(fx, fx), dmul_rn(fy, fy)), r2);
  const double disc = dsub_rn(dmul_rn(b, b), c);
  if (!(disc >= 0.0)) return __longlong_as_double(0x7ff0000000000000LL);
  const double sq = sqrt(disc);
  const double t1 = dsub_rn(-b, sq), t2 = dadd_rn(-b, sq);
  if (t1 > 1e-9) return t1;
  if (t2 > 1e-9) return t2;
  return __longlong_as_double(0x7ff0000000000000LL);
}

// ---------------------------------------------------------------------------
// simple_spread (scenarios/simple_spread.py): NA agents (dyn rows 0..NA-1),
// NA markers (stat rows 0..NA-1). Pairs: agent-agent, lexicographic.
// sc[0] = f32 touching threshold (r_a + r_b), sc[1] = f32(collision_penalty)
// ---------------------------------------------------------------------------
// One env of simple_spread, in registers; shared by the eager kernel and the
// bulk-copy pipeline so both run the same arithmetic.
template <int NA>
struct SpreadEnv {
  static constexpr int O = 4 * NA + 2;
  float px[NA], py[NA], vx[NA], vy[NA], mx[NA], my[NA];

  // decode + contacts (lexicographic pair order) + integrate, once per
  // physics sub-step (PhysK.substeps; the decoded actions are held)
  SS_DEV void physics(const float2 (&u)[NA], const SmallArgs& a) {
    float ux[NA], uy[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const SsEntityDesc& d = a.ents[i];
      ux[i] = decode_axis(u[i].x, d, a.raw_forces);
      uy[i] = decode_axis(u[i].y, d, a.raw_forces);
      if (a.ph.has_gravity) { ux[i] = fadd(ux[i], d.grav_x); uy[i] = fadd(uy[i], d.grav_y); }
    }
    for (int sub = 0; sub < a.ph.substeps; ++sub) {
      float fx[NA], fy[NA];
#pragma unroll
      for (int i = 0; i < NA; ++i) { fx[i] = ux[i]; fy[i] = uy[i]; }
      int p = 0;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
#pragma unroll
        for (int j = i + 1; j < NA; ++j, ++p) {
          const SsPairDesc pr = a.pairs[p];
          float cx, cy;
          if (contact_force(px[i], py[i], px[j], py[j], pr.d_min, pr.d2_act, pr.sign, a.ph.ck, a.ph.k, cx, cy)) {
            fx[i] = fadd(fx[i], cx); fy[i] = fadd(fy[i], cy);
            fx[j] = fsub(fx[j], cx); fy[j] = fsub(fy[j], cy);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const SsEntityDesc& d = a.ents[i];
        integrate_lin(px[i], py[i], vx[i], vy[i], fx[i], fy[i], a.ph.keep, d.inv_m_dt, a.ph.dt,
                      d.max_speed);
      }
    }
  }

  // simple_spread.py:39-46: -(sum over markers of the nearest agent, float64)
  // - penalty * #teammates touching.  min distance = sqrt(min squared distance).
  SS_DEV void rewards(const SmallArgs& a, float (&rew)[NA]) const {
    const float pen = a.sc[1], thr2 = a.sc[2];
    double cover = 0.0;
#pragma unroll
    for (int m = 0; m < NA; ++m) {
      float best = sqnorm(fsub(px[0], mx[m]), fsub(py[0], my[m]));
#pragma unroll
      for (int i = 1; i < NA; ++i) best = fminf(best, sqnorm(fsub(px[i], mx[m]), fsub(py[i], my[m])));
      cover = dadd_rn(cover, (double)fsqrt(best));
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      float coll = 0.0f;
#pragma unroll
      for (int o = 0; o < NA; ++o) {
        if (o == i) continue;
        coll = fadd(coll, sqnorm(fsub(px[i], px[o]), fsub(py[i], py[o])) <= thr2 ? 1.0f : 0.0f);
      }
      rew[i] = (float)dsub_rn(-cover, (double)fmul(pen, coll));
    }
  }

  // simple_spread.py:48-54: [x, y, vx, vy, (marker - self), (other - self)]
  SS_DEV void obs_row(int i, float* row) const {
    row[0] = px[i]; row[1] = py[i]; row[2] = vx[i]; row[3] = vy[i];
    int c = 4;
#pragma unroll
    for (int m = 0; m < NA; ++m) { row[c++] = fsub(mx[m], px[i]); row[c++] = fsub(my[m], py[i]); }
#pragma unroll
    for (int o = 0; o < NA; ++o) {
      if (o == i) continue;
      row[c++] = fsub(px[o], px[i]); row[c++] = fsub(py[o], py[i]);
    }
  }
};

template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_simple_spread(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = SpreadEnv<NA>::O;
  const int64_t B = a.s.B;
  const int64_t e = a.e_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  SpreadEnv<NA> v;
  float2 u[NA];
  int64_t steps = 0;
  if (valid) {
    // every global load of the step issued up front
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const float4 q = a.s.dyn[i * B + e];
      v.px[i] = q.x; v.py[i] = q.y; v.vx[i] = q.z; v.vy[i] = q.w;
      const float2 m = a.s.stat[i * B + e];
      v.mx[i] = m.x; v.my[i] = m.y;
    }
    if (a.mode & SS_DO_PHYSICS) {
#pragma unroll
      for (int i = 0; i < NA; ++i) u[i] = a.act[i][e];
    }
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
  }
  if (valid && (a.mode & SS_DO_PHYSICS)) {
    v.physics(u, a);
#pragma unroll
    for (int i = 0; i < NA; ++i) a.s.dyn[i * B + e] = make_float4(v.px[i], v.py[i], v.vx[i], v.vy[i]);
  }
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; a.s.step_count[e] = steps; }
  if (valid && (a.mode & SS_DO_REWARD)) {
    float rew[NA];
    v.rewards(a, rew);
#pragma unroll
    for (int i = 0; i < NA; ++i) __stcs(a.rew + i * B + e, rew[i]);
  }
  if (valid && (a.mode & SS_DO_DONE)) a.done[e] = (uint8_t)(steps >= a.ph.max_steps);
  if (a.mode & SS_DO_OBS) {
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) v.obs_row(i, row);
      if (nvalid > 0) warp_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
}

// ---------------------------------------------------------------------------
// simple_spread, persistent bulk-copy pipeline (full Env.step mode only).
// Each CTA walks tiles of 128 consecutive envs; the next tile's inputs
// (agent rows, marker rows, actions, step_count — all contiguous spans) are
// prefetched with cp.async.bulk into the other half of a double buffer
// while the current tile computes; outputs are staged in shared memory and
// written back with bulk stores (observations: one contiguous span per
// agent per tile).  The arithmetic is SpreadEnv's, identical to the eager
// kernel.
// ---------------------------------------------------------------------------
constexpr int kPipeTile = 128;
constexpr int kPipeStages = 4;     // input tiles in flight per CTA
constexpr int kPipeOut = 2;        // output staging buffers per CTA

template <int NA>
struct PipeSmem {
  float4 dyn[kPipeStages][NA][kPipeTile];
  float2 stat[kPipeStages][NA][kPipeTile];
  float2 act[kPipeStages][NA][kPipeTile];
  int64_t steps[kPipeStages][kPipeTile];
  float4 dyn_o[kPipeOut][NA][kPipeTile];
  float obs[kPipeOut][NA][kPipeTile * SpreadEnv<NA>::O];
  float rew[kPipeOut][NA][kPipeTile];
  int64_t steps_o[kPipeOut][kPipeTile];
  uint8_t done[kPipeOut][kPipeTile];
  uint64_t bar[kPipeStages];
};

template <int NA>
__global__ void __launch_bounds__(kPipeTile) k_simple_spread_pipe(const SmallArgs a, int64_t ntiles) {
  extern __shared__ __align__(16) float smem_pipe[];
  PipeSmem<NA>& S = *reinterpret_cast<PipeSmem<NA>*>(smem_pipe);
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = SpreadEnv<NA>::O;
  const int tid = threadIdx.x;
  const int64_t B = a.s.B;
  constexpr uint32_t kTileBytes = NA * kPipeTile * (16 + 8 + 8) + kPipeTile * 8;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kPipeStages; ++s) mbar_init(&S.bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int64_t t, int s) {
    const int64_t e0 = t * kPipeTile;
    mbar_arrive_expect_tx(&S.bar[s], kTileBytes);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      bulk_load(&S.dyn[s][i][0], a.s.dyn + i * B + e0, kPipeTile * 16, &S.bar[s]);
      bulk_load(&S.stat[s][i][0], a.s.stat + i * B + e0, kPipeTile * 8, &S.bar[s]);
      bulk_load(&S.act[s][i][0], a.act[i] + e0, kPipeTile * 8, &S.bar[s]);
    }
    bulk_load(&S.steps[s][0], a.s.step_count + e0, kPipeTile * 8, &S.bar[s]);
  };
  int64_t t = blockIdx.x;
  if (tid == 0) {   // prologue: fill kPipeStages - 1 stages
#pragma unroll
    for (int k = 0; k < kPipeStages - 1; ++k)
      if (t + (int64_t)k * gridDim.x < ntiles) issue(t + (int64_t)k * gridDim.x, k);
  }
  for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % kPipeStages;
    const int o = it % kPipeOut;
    // refill the stage consumed in the previous iteration (all threads passed
    // its trailing __syncthreads, so its inputs are dead)
    const int64_t tn = t + (int64_t)(kPipeStages - 1) * gridDim.x;
    if (tn < ntiles && tid == 0) issue(tn, (it + kPipeStages - 1) % kPipeStages);
    mbar_wait(&S.bar[s], (it / kPipeStages) & 1);
    SpreadEnv<NA> v;
    float2 u[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const float4 q = S.dyn[s][i][tid];
      v.px[i] = q.x; v.py[i] = q.y; v.vx[i] = q.z; v.vy[i] = q.w;
      const float2 m = S.stat[s][i][tid];
      v.mx[i] = m.x; v.my[i] = m.y;
      u[i] = S.act[s][i][tid];
    }
    const int64_t steps = S.steps[s][tid] + 1;
    v.physics(u, a);
    float rew[NA];
    v.rewards(a, rew);
    // output buffer o was last used kPipeOut iterations ago: allow the most
    // recent kPipeOut - 1 store groups to still be reading
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kPipeOut - 1) : "memory");
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      S.dyn_o[o][i][tid] = make_float4(v.px[i], v.py[i], v.vx[i], v.vy[i]);
      S.rew[o][i][tid] = rew[i];
      v.obs_row(i, &S.obs[o][i][tid * O]);
    }
    S.steps_o[o][tid] = steps;
    S.done[o][tid] = (uint8_t)(steps >= a.ph.max_steps);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const int64_t e0 = t * kPipeTile;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        bulk_store(a.obs + i * a.obs_stride + e0 * O, &S.obs[o][i][0], kPipeTile * O * 4);
        bulk_store(a.s.dyn + i * B + e0, &S.dyn_o[o][i][0], kPipeTile * 16);
        bulk_store(a.rew + i * B + e0, &S.rew[o][i][0], kPipeTile * 4);
      }
      bulk_store(a.s.step_count + e0, &S.steps_o[o][0], kPipeTile * 8);
      bulk_store(a.done + e0, &S.done[o][0], kPipeTile);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
}

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
template <int NA, int REV>
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
    const double hx = a.sd[0], hy = a.sd[1];
    float ux[NA + 1], uy[NA + 1];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const SsEntityDesc& d = a.ents[i];
      ux[i] = decode_axis(u[i].x, d, a.raw_forces);
      uy[i] = decode_axis(u[i].y, d, a.raw_forces);
    }
    ux[NA] = 0.0f; uy[NA] = 0.0f;
    if (a.ph.has_gravity) {
#pragma unroll
      for (int i = 0; i <= NA; ++i) {
        ux[i] = fadd(ux[i], a.ents[i].grav_x); uy[i] = fadd(uy[i], a.ents[i].grav_y);
      }
    }
    for (int sub = 0; sub < a.ph.substeps; ++sub) {   // physics sub-steps (1 = reference)
      float fx[NA + 1], fy[NA + 1];
#pragma unroll
      for (int i = 0; i <= NA; ++i) { fx[i] = ux[i]; fy[i] = uy[i]; }
      int p = 0;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
#pragma unroll
        for (int j = i + 1; j < NA; ++j, ++p) {
          const SsPairDesc pr = a.pairs[p];
          float cx, cy;
          if (contact_force(px[i], py[i], px[j], py[j], pr.d_min, pr.d2_act, pr.sign, a.ph.ck, a.ph.k, cx, cy)) {
            fx[i] = fadd(fx[i], cx); fy[i] = fadd(fy[i], cy);
            fx[j] = fsub(fx[j], cx); fy[j] = fsub(fy[j], cy);
          }
        }
        {  // agent i vs package (sphere-box)
          const SsPairDesc pr = a.pairs[p++];
          float qx, qy, cx, cy;
          closest_point_on_box(px[i], py[i], px[NA], py[NA], ca, sa, hx, hy, qx, qy);
          if (contact_force(px[i], py[i], qx, qy, pr.d_min, pr.d2_act, pr.sign, a.ph.ck, a.ph.k, cx, cy)) {
            fx[i] = fadd(fx[i], cx); fy[i] = fadd(fy[i], cy);
            fx[NA] = fsub(fx[NA], cx); fy[NA] = fsub(fy[NA], cy);
          }
        }
      }
#pragma unroll
      for (int i = 0; i <= NA; ++i) {
        const SsEntityDesc& d = a.ents[i];
        integrate_lin(px[i], py[i], vx[i], vy[i], fx[i], fy[i], a.ph.keep, d.inv_m_dt, a.ph.dt,
                      d.max_speed);
      }
    }
#pragma unroll
    for (int i = 0; i <= NA; ++i) a.s.dyn[i * B + e] = make_float4(px[i], py[i], vx[i], vy[i]);
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
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) {
        row[0] = px[i]; row[1] = py[i]; row[2] = vx[i]; row[3] = vy[i];
        row[4] = fsub(px[NA], px[i]); row[5] = fsub(py[NA], py[i]);
        if (REV) {
          row[6] = vx[NA]; row[7] = vy[NA];
          row[8] = fsub(gx, px[NA]); row[9] = fsub(gy, py[NA]);
        } else {
          row[6] = fsub(gx, px[i]); row[7] = fsub(gy, py[i]);
          row[8] = fsub(px[NA], gx); row[9] = fsub(py[NA], gy);
          row[10] = vx[NA]; row[11] = vy[NA];
        }
      }
      if (nvalid > 0) warp_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
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
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * O);
    float* row = sbuf + (threadIdx.x & 31) * O;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
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
      if (nvalid > 0) warp_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, O, sbuf);
    }
  }
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
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_wheel(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 10;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
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
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_give_way(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 12;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
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
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_passage(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 10 + 2 * (NA - 1);
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
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
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_balance(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int O = 17;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
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
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_waterfall(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  const int NB = a.si[2];
  const int O = a.obs_dim;   // 6 + 2 NB
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
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
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_football(const SmallArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  constexpr int NT = NA / 2;
  constexpr int O = 4 + 2 + 2 + 2 * (NA - 1) + 2;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
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

// ---------------------------------------------------------------------------
// flocking (scenarios/flocking.py): NA agents (dyn 0..NA-1), beacon marker
// (entity NA, stat row 0), NO rocks (entity NA+1+r, stat row 1+r, immovable).
// Pairs, lexicographic: for i: agents j>i, then rocks.  Optional Lidar
// (sensors.py) appended to the observation: n_rays ranges per agent.
// sc[0] = f32 agent-agent touch threshold, sc[1] = agent-rock threshold,
// sc[2] = f32(collision_penalty); si[4] = NO; sd[0], sd[1] = agent / rock
// radius^2 as python doubles (sensors.py:47).
// ---------------------------------------------------------------------------
// Conservative float32 screen of one (ray, circle) pair.  It returns false
// only when the exact float64 test (ray_circle, sensors.py:43-54) is certain
// to yield no hit or a hit beyond max_range — i.e. when skipping the pair
// cannot change min(best, max_range).  Every surviving pair is evaluated in
// float64 exactly as the reference, so the lidar output stays bit-identical.
// Margins (1e-4) dominate the float32 rounding of these few products by
// more than two orders of magnitude for |origin - centre| up to ~1e2; pairs
// farther than max_range are rejected by the first test before that.
struct RayScreen {
  float rr;       // r + 1e-4
  float reach2;   // (max_range + r + 1e-4)^2
  float r2;       // r^2 (float32)
};

SS_DEV bool ray_may_hit(float fx, float fy, float dx, float dy, const RayScreen& s) {
  const float f2 = fx * fx + fy * fy;
  if (!(f2 <= s.reach2)) return false;       // every hit lies beyond max_range
  const float cr = fx * dy - fy * dx;
  if (fabsf(cr) > s.rr) return false;        // line misses the circle
  const float b = fx * dx + fy * dy;
  if (b > 1e-4f && f2 - s.r2 > 1e-4f) return false;   // circle behind an outside origin
  return true;
}

// Screen all rays against one circle: bit m set when ray m may hit.
SS_DEV uint32_t ray_mask(float fx, float fy, const float2* dirs, int n_rays, const RayScreen& s) {
  const float f2 = fx * fx + fy * fy;
  if (!(f2 <= s.reach2)) return 0u;
  const bool outside = f2 - s.r2 > 1e-4f;
  uint32_t mask = 0u;
  for (int m = 0; m < n_rays; ++m) {
    const float2 d = dirs[m];
    const float cr = fx * d.y - fy * d.x;
    const float b = fx * d.x + fy * d.y;
    const bool may = fabsf(cr) <= s.rr && !(outside && b > 1e-4f);
    mask |= (uint32_t)may << m;
  }
  return mask;
}

// Exact float64 tests for the screened-in rays of one circle; per-ray minima
// live in shared memory (best[m * kSmallThreads]), so the divergent work is
// proportional to the number of surviving (ray, circle) pairs, not n_rays.
SS_DEV void ray_hits(uint32_t mask, double ox, double oy, const double* dir_table, double cx,
                     double cy, double r2, double* best, int stride = kSmallThreads) {
  while (mask) {
    const int m = __ffs(mask) - 1;
    mask &= mask - 1u;
    const double t = ray_circle(ox, oy, dir_table[2 * m], dir_table[2 * m + 1], cx, cy, r2);
    best[m * stride] = fmin(best[m * stride], t);
  }
}

// Uniform ray fan (sensors.py:40-43): angle_m = start + m * step, m < n,
// with 0 < n * step <= 2 pi.  All quantities in units of `step`.
struct RayFan {
  float start;      // start angle (rad)
  float inv_step;   // 1 / step
  float period;     // 2 pi / step
  float quarter;    // (pi / 2) / step
  uint32_t all;     // bits 0..n-1
  int n;
  int full;         // span == 2 pi: period == n, windows wrap by rotation
};

// atan2 with |error| < 2e-6 rad over all quadrants (checked on the host
// against libm atan2 on 2e7 angles); minimax polynomial on [0, 1].
SS_DEV float fast_atan2(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float t = mx > 0.f ? __fdividef(mn, mx) : 0.f;
  const float s = __fmul_rn(t, t);
  float p = -0.01172120f;
  p = __fmaf_rn(p, s, 0.05265332f);
  p = __fmaf_rn(p, s, -0.11643287f);
  p = __fmaf_rn(p, s, 0.19354346f);
  p = __fmaf_rn(p, s, -0.33262347f);
  p = __fmaf_rn(p, s, 0.99997726f);
  float r = __fmul_rn(p, t);
  if (ay > ax) r = __fsub_rn(1.57079637f, r);
  if (x < 0.f) r = __fsub_rn(3.14159274f, r);
  return copysignf(r, y);
}

// Rays m (0 <= m < n) with lo <= m <= hi.
SS_DEV uint32_t ray_bits(float lo, float hi, int n) {
  const int a = max((int)ceilf(fmaxf(lo, -1.0f)), 0);
  const int b = min((int)floorf(fminf(hi, 64.0f)), n - 1);
  if (a > b) return 0u;
  return (0xffffffffu >> (31 - b)) & (0xffffffffu << a);
}

// Conservative angular screen of one circle against a whole fan: a ray can
// hit a circle of radius r seen at distance |f| > r only if its angle lies
// within asin(r / |f|) <= r / sqrt(|f|^2 - r^2) of the bearing to the centre
// (and then it points towards it).  The window is widened by 0.1% + 0.01
// ray spacings (>= 2.5e3 x the atan2 / rsqrt / fp32 rounding error) and r by
// 1e-4, so every ray the exact float64 test could report within max_range
// is kept; origins on or inside the (widened) rim and windows wider than
// pi/2 keep every ray.
SS_DEV uint32_t ray_window(float fx, float fy, const RayFan& fan, const RayScreen& s) {
  const float f2 = __fadd_rn(__fmul_rn(fx, fx), __fmul_rn(fy, fy));
  if (!(f2 <= s.reach2)) return 0u;
  const float q = __fsub_rn(f2, __fmul_rn(s.rr, s.rr));
  if (!(q > 1e-6f)) return fan.all;
#ifdef SS_TEST_SHRINK_FAN   // deliberately broken screen: tests must catch it
  const float w = 0.97f * __fmul_rn(__fmul_rn(s.rr, rsqrtf(q)), fan.inv_step);
#else
  const float w = __fmaf_rn(__fmul_rn(__fmul_rn(s.rr, rsqrtf(q)), fan.inv_step), 1.001f, 0.01f);
#endif
  if (!(w < fan.quarter)) return fan.all;
  float v = __fmul_rn(__fsub_rn(fast_atan2(-fy, -fx), fan.start), fan.inv_step);
  v = __fsub_rn(v, __fmul_rn(fan.period, floorf(__fdividef(v, fan.period))));
  if (fan.full) {
    // rays lo..hi modulo n: one contiguous run rotated into place
    const int lo = (int)ceilf(v - w), hi = (int)floorf(v + w);   // -n/4 <= lo, hi < 5n/4
    const int cnt = hi - lo + 1;
    if (cnt <= 0) return 0u;
    if (cnt >= fan.n) return fan.all;
    const int base = lo < 0 ? lo + fan.n : (lo >= fan.n ? lo - fan.n : lo);
    const uint64_t m = (uint64_t)((1u << cnt) - 1u) << base;
    return (uint32_t)(m | (m >> fan.n)) & fan.all;
  }
  return ray_bits(v - w, v + w, fan.n) | ray_bits(v - w + fan.period, v + w + fan.period, fan.n) |
         ray_bits(v - w - fan.period, v + w - fan.period, fan.n);
}

// ray_hits with the minima kept as float bits (see lidar_fan_warp).
SS_DEV void ray_hits_f(uint32_t mask, double ox, double oy, const double2* dirs, double cx, double cy,
                       double r2, uint32_t* best, int stride) {
  while (mask) {
    const int m = __ffs(mask) - 1;
    mask &= mask - 1u;
    const double t = ray_circle(ox, oy, dirs[m].x, dirs[m].y, cx, cy, r2);
    best[m * stride] = min(best[m * stride], __float_as_uint((float)t));
  }
}

struct FlockLidarK {
  double r2_agent, r2_rock;
  RayScreen agent, rock;
  RayFan fan;
  int fan_ok;   // uniform fan usable (else the per-ray screen)
};

constexpr int kLidarQueue = 64;    // (lane, target, ray) tests staged per warp and round

// Lidar of agent i for the 32 envs of one warp (k_flocking_w), load-balanced
// across lanes: each lane screens its env's targets with ray_window, the
// surviving (env, target, ray) triples are compacted into a per-warp queue
// (warp prefix sum) and the exact float64 tests are dealt out 32 at a time,
// so a warp runs ceil(total / 32) test rounds instead of the maximum per-lane
// count per target.  Minima land in the staged observation rows themselves
// (best[lane * P + ray], the lidar columns) as float bits (atomicMin on
// the non-negative float pattern): float(min(t, range)) == min(float(t),
// float(range)) since rounding is monotone, so the scan stays bit-identical.
// Warp-collective: every lane of the warp must call it.
template <int NA>
SS_DEV void lidar_fan_warp(bool active, int i, int lane, int NO, float mex, float mey,
                           const float2* spos, const float2* sst, const FlockLidarK& lk,
                           const double2* sdird, uint32_t* best, int P, uint32_t* queue, int n_rays) {
  constexpr int NT = NA - 1 + kFlockMaxRocks;
  uint32_t mk[NT];
  int cnt = 0;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    mk[t] = 0u;
    if (active && (t < NA - 1 || t - (NA - 1) < NO)) {
      float qx, qy;
      if (t < NA - 1) {
        const float2 q = spos[(t < i ? t : t + 1) * 32 + lane];
        qx = q.x; qy = q.y;
      } else {
        const float2 q = sst[(t - (NA - 1) + 1) * 32 + lane];
        qx = q.x; qy = q.y;
      }
      mk[t] = ray_window(__fsub_rn(mex, qx), __fsub_rn(mey, qy), lk.fan, t < NA - 1 ? lk.agent : lk.rock);
      cnt += __popc(mk[t]);
    }
  }
  for (int m = 0; m < n_rays; ++m) best[lane * P + m] = 0x7f800000u;   // +inf
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  const int excl = incl - cnt;
  for (int base = 0; base < total; base += kLidarQueue) {
    if (excl < base + kLidarQueue && excl + cnt > base) {
      int idx = excl;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        uint32_t m = mk[t];
        while (m) {
          const int r = __ffs(m) - 1;
          m &= m - 1u;
          if (idx >= base && idx < base + kLidarQueue) queue[idx - base] = (uint32_t)lane | (t << 5) | (r << 9);
          ++idx;
        }
      }
    }
    __syncwarp();
    const int nq = min(kLidarQueue, total - base);
    for (int k = lane; k < nq; k += 32) {
      const uint32_t w = queue[k];
      const int sl = (int)(w & 31u), t = (int)((w >> 5) & 15u), r = (int)(w >> 9);
      const float2 org = spos[i * 32 + sl];
      double cx, cy, r2;
      if (t < NA - 1) {
        const float2 q = spos[(t < i ? t : t + 1) * 32 + sl];
        cx = q.x; cy = q.y; r2 = lk.r2_agent;
      } else {
        const float2 q = sst[(t - (NA - 1) + 1) * 32 + sl];
        cx = q.x; cy = q.y; r2 = lk.r2_rock;
      }
      const double2 d = sdird[r];
      const double tt = ray_circle((double)org.x, (double)org.y, d.x, d.y, cx, cy, r2);
      if (tt < __longlong_as_double(0x7ff0000000000000LL))
        atomicMin(best + sl * P + r, __float_as_uint((float)tt));
    }
    __syncwarp();
  }
}

inline RayScreen make_screen(double r, double max_range) {
  RayScreen s;
  s.rr = (float)r + 1e-4f;
  const float reach = (float)max_range + s.rr;
  s.reach2 = reach * reach;
  s.r2 = (float)(r * r);
  return s;
}

template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_SMALL_MINB) k_flocking(const SmallArgs a, const FlockLidarK lk) {
  extern __shared__ __align__(16) float smem_raw[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  const int NO = a.si[4];
  const int O = a.obs_dim;
  // shared memory: [per-ray best hits: n_rays x kSmallThreads doubles]
  //                [float32 ray directions: n_rays (padded to even) float2]
  //                [per-warp obs staging: kSmallThreads x O floats]
  double* sbest = reinterpret_cast<double*>(smem_raw);
  float2* sdir = reinterpret_cast<float2*>(sbest + a.n_rays * kSmallThreads);
  float* smem = reinterpret_cast<float*>(sdir + ((a.n_rays + 1) & ~1));
  if (threadIdx.x < a.n_rays)
    sdir[threadIdx.x] = make_float2((float)a.ray_dir[2 * threadIdx.x], (float)a.ray_dir[2 * threadIdx.x + 1]);
  __syncthreads();
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  float px[NA], py[NA], vx[NA], vy[NA];
  float rx[kFlockMaxRocks], ry[kFlockMaxRocks];
  float bx = 0.f, by = 0.f;
  if (valid) {
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const float4 q = a.s.dyn[i * B + e];
      px[i] = q.x; py[i] = q.y; vx[i] = q.z; vy[i] = q.w;
    }
    const float2 bq = a.s.stat[e];
    bx = bq.x; by = bq.y;
#pragma unroll
    for (int r = 0; r < kFlockMaxRocks; ++r) {
      if (r < NO) { const float2 q = a.s.stat[(1 + r) * B + e]; rx[r] = q.x; ry[r] = q.y; }
      else { rx[r] = 0.f; ry[r] = 0.f; }
    }
  }
  if (valid && (a.mode & SS_DO_PHYSICS)) {
    float ux[NA], uy[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const SsEntityDesc& d = a.ents[i];
      const float2 u = a.act[i][e];
      ux[i] = decode_axis(u.x, d, a.raw_forces);
      uy[i] = decode_axis(u.y, d, a.raw_forces);
      if (a.ph.has_gravity) { ux[i] = fadd(ux[i], d.grav_x); uy[i] = fadd(uy[i], d.grav_y); }
    }
    for (int sub = 0; sub < a.ph.substeps; ++sub) {   // physics sub-steps (1 = reference)
    float fx[NA], fy[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) { fx[i] = ux[i]; fy[i] = uy[i]; }
    int p = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
#pragma unroll
      for (int j = i + 1; j < NA; ++j, ++p) {
        const SsPairDesc pr = a.pairs[p];
        float cx, cy;
        if (contact_force(px[i], py[i], px[j], py[j], pr.d_min, pr.d2_act, pr.sign, a.ph.ck, a.ph.k, cx, cy)) {
          fx[i] = fadd(fx[i], cx); fy[i] = fadd(fy[i], cy);
          fx[j] = fsub(fx[j], cx); fy[j] = fsub(fy[j], cy);
        }
      }
#pragma unroll
      for (int r = 0; r < kFlockMaxRocks; ++r) {
        if (r < NO) {
          const SsPairDesc pr = a.pairs[p++];
          float cx, cy;
          if (contact_force(px[i], py[i], rx[r], ry[r], pr.d_min, pr.d2_act, pr.sign, a.ph.ck, a.ph.k, cx, cy)) {
            fx[i] = fadd(fx[i], cx); fy[i] = fadd(fy[i], cy);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const SsEntityDesc& d = a.ents[i];
      integrate_lin(px[i], py[i], vx[i], vy[i], fx[i], fy[i], a.ph.keep, d.inv_m_dt, a.ph.dt,
                    d.max_speed);
    }
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) a.s.dyn[i * B + e] = make_float4(px[i], py[i], vx[i], vy[i]);
  }
  int64_t steps = 0;
  if (valid && (a.mode & (SS_DO_COUNT | SS_DO_DONE))) {
    steps = a.s.step_count[e];
    if (a.mode & SS_DO_COUNT) { steps += 1; a.s.step_count[e] = steps; }
  }
  if (valid && (a.mode & SS_DO_REWARD)) {
    const float pen = a.sc[2], thr2_aa = a.sc[3], thr2_ar = a.sc[4];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const float gap = norm2(fsub(px[i], bx), fsub(py[i], by));
      float ca = 0.0f, cr = 0.0f;
#pragma unroll
      for (int o = 0; o < NA; ++o) {
        if (o == i) continue;
        ca = fadd(ca, sqnorm(fsub(px[i], px[o]), fsub(py[i], py[o])) <= thr2_aa ? 1.0f : 0.0f);
      }
#pragma unroll
      for (int r = 0; r < kFlockMaxRocks; ++r) {
        if (r < NO) cr = fadd(cr, sqnorm(fsub(px[i], rx[r]), fsub(py[i], ry[r])) <= thr2_ar ? 1.0f : 0.0f);
      }
      __stcs(a.rew + i * B + e, fsub(-gap, fmul(pen, fadd(ca, cr))));
    }
  }
  if (valid && (a.mode & SS_DO_DONE)) a.done[e] = (uint8_t)(steps >= a.ph.max_steps);
  if (a.mode & SS_DO_OBS) {
    const int P = O | 1;   // odd per-lane stride: conflict-free row writes
    float* sbuf = smem + (threadIdx.x >> 5) * (32 * P);
    float* row = sbuf + (threadIdx.x & 31) * P;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (valid) {
        row[0] = px[i]; row[1] = py[i]; row[2] = vx[i]; row[3] = vy[i];
        row[4] = fsub(bx, px[i]); row[5] = fsub(by, py[i]);
        int c = 6;
#pragma unroll
        for (int r = 0; r < kFlockMaxRocks; ++r) {
          if (r < NO) { row[c] = fsub(rx[r], px[i]); row[c + 1] = fsub(ry[r], py[i]); c += 2; }
        }
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          if (o == i) continue;
          row[c] = fsub(px[o], px[i]); row[c + 1] = fsub(py[o], py[i]); c += 2;
        }
        if (a.n_rays > 0) {
          // lidar_scan (sensors.py:138-146): fp64 rays vs every collidable
          // entity except the emitter; nearest hit, capped at max_range.
          const double ox = (double)px[i], oy = (double)py[i];
          const float rot_i = a.attach_rot ? a.s.rot[i * B + e].x : 0.0f;
          if (rot_i == 0.0f) {
            double* best = sbest + threadIdx.x;
            for (int m = 0; m < a.n_rays; ++m) best[m * kSmallThreads] = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
            for (int o = 0; o < NA; ++o) {
              if (o == i) continue;
              const uint32_t mk = ray_mask(px[i] - px[o], py[i] - py[o], sdir, a.n_rays, lk.agent);
              ray_hits(mk, ox, oy, a.ray_dir, (double)px[o], (double)py[o], lk.r2_agent, best);
            }
#pragma unroll
            for (int r = 0; r < kFlockMaxRocks; ++r) {
              if (r < NO) {
                const uint32_t mk = ray_mask(px[i] - rx[r], py[i] - ry[r], sdir, a.n_rays, lk.rock);
                ray_hits(mk, ox, oy, a.ray_dir, (double)rx[r], (double)ry[r], lk.r2_rock, best);
              }
            }
            for (int m = 0; m < a.n_rays; ++m) row[c + m] = (float)fmin(best[m * kSmallThreads], a.lidar_range);
          } else
          for (int m = 0; m < a.n_rays; ++m) {
            double dx, dy;
            if (rot_i == 0.0f) { dx = a.ray_dir[2 * m]; dy = a.ray_dir[2 * m + 1]; }
            else {
              const double ang = dadd_rn(dadd_rn(a.ray_start, (double)m * a.ray_span / a.n_rays),
                                      (double)rot_i);
              sincos(ang, &dy, &dx);
            }
            const float dx32 = (float)dx, dy32 = (float)dy;
            double best = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
            for (int o = 0; o < NA; ++o) {
              if (o == i) continue;
              if (ray_may_hit(px[i] - px[o], py[i] - py[o], dx32, dy32, lk.agent))
                best = fmin(best, ray_circle(ox, oy, dx, dy, (double)px[o], (double)py[o], lk.r2_agent));
            }
#pragma unroll
            for (int r = 0; r < kFlockMaxRocks; ++r) {
              if (r < NO && ray_may_hit(px[i] - rx[r], py[i] - ry[r], dx32, dy32, lk.rock))
                best = fmin(best, ray_circle(ox, oy, dx, dy, (double)rx[r], (double)ry[r], lk.r2_rock));
            }
            row[c + m] = (float)fmin(best, a.lidar_range);
          }
        }
      }
      if (nvalid > 0) warp_flush_padded(a.obs + i * a.obs_stride + e0 * O, nvalid, O, P, sbuf);
    }
  }
}

// ---------------------------------------------------------------------------
// flocking, warp-per-agent mapping: a CTA of NA warps handles 32 envs; warp
// i owns agent i of those envs (lane = env).  Each thread sums the force on
// its own agent over the reference's pair order restricted to that agent —
// (j, i) for j < i subtracted, then (i, j) for agents j > i and the rocks
// added (dynamics.py:163-180) — reading partners from shared memory, then
// builds agent i's reward, observation row and lidar scan.  NA x more
// threads per env than k_flocking: the 100k-env config fills the GPU.
// sc[5] = f32 agent-agent d_min, sc[6] its squared bound, sc[7] agent-rock
// d_min, sc[8] its squared bound (uniform radii are a template condition).
// ---------------------------------------------------------------------------
#ifndef SS_FLOCK_WARPS
#define SS_FLOCK_WARPS 40   // resident warps per SM the register budget is sized for
#endif
template <int NA>
__global__ void __launch_bounds__(32 * NA, (SS_FLOCK_WARPS / NA < 32 ? SS_FLOCK_WARPS / NA : 32))
    k_flocking_w(const SmallArgs a, const FlockLidarK lk) {
  extern __shared__ __align__(16) float smem_w[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  const int NO = a.si[4];
  const int O = a.obs_dim;
  const int P = O | 1;
  const int lane = threadIdx.x & 31, i = threadIdx.x >> 5;
  const int64_t B = a.s.B;
  const int64_t e0 = (int64_t)blockIdx.x * 32;
  const int64_t e = e0 + lane;
  const bool valid = e < B;
  const int nvalid = (int)min((int64_t)32, B - e0);
  // shared memory: [dirs: n_rays double2][agents: NA x 32 float4 pre-step]
  //                [agents: NA x 32 float2 post-step positions][queue: NA x kLidarQueue u32]
  //                [dirs: n_rays(+1) float2][static: (1+NO) x 32 float2][rows: NA warps x 32 x P]
  // (pre / post copies: one barrier between physics and the rest; the lidar
  // minima are accumulated in the rows' lidar columns)
  double2* sdird = reinterpret_cast<double2*>(smem_w);
  float4* sag = reinterpret_cast<float4*>(sdird + a.n_rays);
  float2* spos = reinterpret_cast<float2*>(sag + NA * 32);
  uint32_t* squeue = reinterpret_cast<uint32_t*>(spos + NA * 32);
  float2* sdir = reinterpret_cast<float2*>(squeue + NA * kLidarQueue);
  float2* sst = reinterpret_cast<float2*>(sdir + ((a.n_rays + 1) & ~1));
  float* srow = reinterpret_cast<float*>(sst + (1 + NO) * 32) + i * 32 * P;
  if (threadIdx.x < a.n_rays) {
    const double dx = a.ray_dir[2 * threadIdx.x], dy = a.ray_dir[2 * threadIdx.x + 1];
    sdird[threadIdx.x] = make_double2(dx, dy);
    sdir[threadIdx.x] = make_float2((float)dx, (float)dy);
  }
  float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t steps = 0;
  float2 u = make_float2(0.f, 0.f);
  if (valid) {
    // every global load of the step issued up front
    me = a.s.dyn[i * B + e];
    if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
    if (a.mode & SS_DO_PHYSICS) u = a.act[i][e];
    sag[i * 32 + lane] = me;
    for (int k = i; k < 1 + NO; k += NA) sst[k * 32 + lane] = a.s.stat[k * B + e];
  }
  __syncthreads();
  if (a.mode & SS_DO_PHYSICS) {
    const SsEntityDesc& d = a.ents[i];
    float ux = decode_axis(u.x, d, a.raw_forces), uy = decode_axis(u.y, d, a.raw_forces);
    if (a.ph.has_gravity) { ux = fadd(ux, d.grav_x); uy = fadd(uy, d.grav_y); }
    const float dmin_aa = a.sc[5], d2_aa = a.sc[6], dmin_ar = a.sc[7], d2_ar = a.sc[8];
    for (int sub = 0; sub < a.ph.substeps; ++sub) {   // physics sub-steps (1 = reference)
    if (sub > 0) {   // restage every agent's sub-step state (all threads reach both barriers)
      __syncthreads();
      if (valid) sag[i * 32 + lane] = me;
      __syncthreads();
    }
    if (valid) {
    float fx = ux, fy = uy;
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      if (j == i) continue;
      const float4 q = sag[j * 32 + lane];
      const float sign = ((i + j) & 1) ? -1.0f : 1.0f;
      float cx, cy;
      if (j < i) {
        if (contact_force(q.x, q.y, me.x, me.y, dmin_aa, d2_aa, sign, a.ph.ck, a.ph.k, cx, cy)) {
          fx = fsub(fx, cx); fy = fsub(fy, cy);
        }
      } else {
        if (contact_force(me.x, me.y, q.x, q.y, dmin_aa, d2_aa, sign, a.ph.ck, a.ph.k, cx, cy)) {
          fx = fadd(fx, cx); fy = fadd(fy, cy);
        }
      }
    }
    for (int r = 0; r < NO; ++r) {
      const float2 q = sst[(1 + r) * 32 + lane];
      const float sign = ((i + NA + 1 + r) & 1) ? -1.0f : 1.0f;
      float cx, cy;
      if (contact_force(me.x, me.y, q.x, q.y, dmin_ar, d2_ar, sign, a.ph.ck, a.ph.k, cx, cy)) {
        fx = fadd(fx, cx); fy = fadd(fy, cy);
      }
    }
    integrate_lin(me.x, me.y, me.z, me.w, fx, fy, a.ph.keep, d.inv_m_dt, a.ph.dt, d.max_speed);
    }
    }
    if (valid) a.s.dyn[i * B + e] = me;
  }
  if (valid) spos[i * 32 + lane] = make_float2(me.x, me.y);
  __syncthreads();                       // post-step positions of every agent staged
  if (valid && (a.mode & SS_DO_COUNT)) { steps += 1; if (i == 0) a.s.step_count[e] = steps; }
  const float2 beacon = valid ? sst[lane] : make_float2(0.f, 0.f);
  if (valid && (a.mode & SS_DO_REWARD)) {
    const float pen = a.sc[2], thr2_aa = a.sc[3], thr2_ar = a.sc[4];
    const float gap = norm2(fsub(me.x, beacon.x), fsub(me.y, beacon.y));
    float ca = 0.0f, cr = 0.0f;
#pragma unroll
    for (int o = 0; o < NA; ++o) {
      if (o == i) continue;
      const float2 q = spos[o * 32 + lane];
      ca = fadd(ca, sqnorm(fsub(me.x, q.x), fsub(me.y, q.y)) <= thr2_aa ? 1.0f : 0.0f);
    }
    for (int r = 0; r < NO; ++r) {
      const float2 q = sst[(1 + r) * 32 + lane];
      cr = fadd(cr, sqnorm(fsub(me.x, q.x), fsub(me.y, q.y)) <= thr2_ar ? 1.0f : 0.0f);
    }
    __stcs(a.rew + i * B + e, fsub(-gap, fmul(pen, fadd(ca, cr))));
  }
  if (valid && i == 0 && (a.mode & SS_DO_DONE)) a.done[e] = (uint8_t)(steps >= a.ph.max_steps);
  if (a.mode & SS_DO_OBS) {
    float* row = srow + lane * P;
    if (valid) {
      row[0] = me.x; row[1] = me.y; row[2] = me.z; row[3] = me.w;
      row[4] = fsub(beacon.x, me.x); row[5] = fsub(beacon.y, me.y);
      int c = 6;
      for (int r = 0; r < NO; ++r) {
        const float2 q = sst[(1 + r) * 32 + lane];
        row[c] = fsub(q.x, me.x); row[c + 1] = fsub(q.y, me.y); c += 2;
      }
#pragma unroll
      for (int o = 0; o < NA; ++o) {
        if (o == i) continue;
        const float2 q = spos[o * 32 + lane];
        row[c] = fsub(q.x, me.x); row[c + 1] = fsub(q.y, me.y); c += 2;
      }
    }
    if (a.n_rays > 0) {
      const int c = 6 + 2 * NO + 2 * (NA - 1);
      const double ox = (double)me.x, oy = (double)me.y;
      const float rot_i = (valid && a.attach_rot) ? a.s.rot[i * B + e].x : 0.0f;
      const bool fan = valid && rot_i == 0.0f;
      uint32_t* wbest = reinterpret_cast<uint32_t*>(srow + c);   // this warp's rows, lidar columns
      uint32_t* best = wbest + lane * P;
      const int stride = 1;
      const float range_f = (float)a.lidar_range;
      if (lk.fan_ok) {
        // warp-collective: all lanes, including invalid / rotated ones
        lidar_fan_warp<NA>(fan, i, lane, NO, me.x, me.y, spos, sst, lk, sdird, wbest, P, squeue + i * kLidarQueue,
                           a.n_rays);
        if (fan)
          for (int m = 0; m < a.n_rays; ++m)
            best[m] = __float_as_uint(fminf(__uint_as_float(best[m]), range_f));
      } else if (fan) {
        for (int m = 0; m < a.n_rays; ++m) best[m * stride] = 0x7f800000u;
#pragma unroll
        for (int o = 0; o < NA; ++o) {
          if (o == i) continue;
          const float2 q = spos[o * 32 + lane];
          const uint32_t mk = ray_mask(me.x - q.x, me.y - q.y, sdir, a.n_rays, lk.agent);
          ray_hits_f(mk, ox, oy, sdird, (double)q.x, (double)q.y, lk.r2_agent, best, stride);
        }
        for (int r = 0; r < NO; ++r) {
          const float2 q = sst[(1 + r) * 32 + lane];
          const uint32_t mk = ray_mask(me.x - q.x, me.y - q.y, sdir, a.n_rays, lk.rock);
          ray_hits_f(mk, ox, oy, sdird, (double)q.x, (double)q.y, lk.r2_rock, best, stride);
        }
        for (int m = 0; m < a.n_rays; ++m) best[m] = __float_as_uint(fminf(__uint_as_float(best[m]), range_f));
      }
      if (valid && !fan) {
        // attached rotation (sensors.py:121-135): per-ray fp64 angles
        for (int m = 0; m < a.n_rays; ++m) {
          const double ang = dadd_rn(dadd_rn(a.ray_start, (double)m * a.ray_span / a.n_rays), (double)rot_i);
          double dx, dy;
          sincos(ang, &dy, &dx);
          double b = __longlong_as_double(0x7ff0000000000000LL);
          for (int o = 0; o < NA; ++o) {
            if (o == i) continue;
            const float2 q = spos[o * 32 + lane];
            b = fmin(b, ray_circle(ox, oy, dx, dy, (double)q.x, (double)q.y, lk.r2_agent));
          }
          for (int r = 0; r < NO; ++r) {
            const float2 q = sst[(1 + r) * 32 + lane];
            b = fmin(b, ray_circle(ox, oy, dx, dy, (double)q.x, (double)q.y, lk.r2_rock));
          }
          row[c + m] = (float)fmin(b, a.lidar_range);
        }
      }
    }
    if (nvalid > 0) warp_flush_padded(a.obs + i * a.obs_stride + e0 * O, nvalid, O, P, srow);
  }
}

inline size_t flocking_w_smem(int NA, int NO, int n_rays, int O) {
  return (size_t)n_rays * sizeof(double2) + (size_t)NA * 32 * sizeof(float4) +
         (size_t)NA * 32 * sizeof(float2) + (size_t)NA * kLidarQueue * sizeof(uint32_t) +
         (size_t)((n_rays + 1) & ~1) * sizeof(float2) + (size_t)(1 + NO) * 32 * sizeof(float2) +
         (size_t)NA * 32 * (O | 1) * sizeof(float);
}

// ---------------------------------------------------------------------------
// Host-side dispatch
// ---------------------------------------------------------------------------
// The bulk-copy pipeline is opt-in (SS_PIPE=1): measured on B200 at 1M envs
// it reaches 68 us/step (4 stages, 2 CTAs/SM) against 60 us for the eager
// register kernel — the per-env arithmetic is latency-bound and the eager
// kernel keeps ~24 warps/SM in flight, the smem-staged pipeline ~8.
// It needs every per-tile span 16-byte aligned: rows of B float2 / float
// entries start at row * B * 8 / row * B * 4 bytes.
static bool pipe_eligible(const World& w, const SmallArgs& a, int NA) {
  static const bool enabled = std::getenv("SS_PIPE") != nullptr;
  if (!enabled || a.mode != SS_MODE_STEP || NA < 2 || NA > 4) return false;
  const int64_t B = w.d.batch;
  if (B < kPipeTile || (B % 4) != 0 || (a.obs_stride % 4) != 0) return false;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  for (int i = 0; i < NA; ++i)
    if (!al(a.act[i])) return false;
  return al(a.s.dyn) && al(a.s.stat) && al(a.s.step_count) && al(a.obs) && al(a.rew) && al(a.done);
}

template <int NA>
static int launch_pipe(World& w, const SmallArgs& a, int64_t ntiles, cudaStream_t st) {
  const size_t smem = sizeof(PipeSmem<NA>);
  static int grid_cap = 0;   // per instantiation: SMs x resident CTAs
  if (grid_cap == 0) {
    cudaFuncSetAttribute(k_simple_spread_pipe<NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_simple_spread_pipe<NA>, kPipeTile, smem);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const unsigned grid = (unsigned)(ntiles < grid_cap ? ntiles : grid_cap);
  if (grid == 0) return SS_OK;
  k_simple_spread_pipe<NA><<<grid, kPipeTile, smem, st>>>(a, ntiles);
  return cuda_status(cudaGetLastError(), "pipelined step launch");
}

int launch_small(World& w, const SsBuffers* buf, const SsStepIO* io, cudaStream_t st) {
  SmallArgs a;
  memset(&a, 0, sizeof(a));
  a.s = make_state(w, buf);
  a.ph = make_phys(w);
  a.ents = w.d_ents;
  a.pairs = w.d_pairs;
  const int NA = w.d.n_agents;
  if (NA < 1 || NA > kSmallMaxAgents) {
    set_error("fused kernel instantiated for 1.." + std::to_string(kSmallMaxAgents) + " agents");
    return SS_ERR_UNSUPPORTED;
  }
  if (io->mode & SS_DO_PHYSICS) {
    for (int i = 0; i < NA; ++i) a.act[i] = reinterpret_cast<const float2*>(io->actions[i]);
  }
  a.obs = io->obs;
  a.obs_stride = io->obs_agent_stride;
  a.rew = io->rew;
  a.done = io->done;
  a.mode = io->mode;
  a.raw_forces = io->raw_forces;
  a.obs_dim = w.d.obs_dim;
  a.guard = io->guard;
  a.guard_n = io->guard_count > 0 ? io->guard_count : 1;
  memcpy(a.sc, w.d.sc, sizeof(a.sc));
  memcpy(a.sd, w.d.sd, sizeof(a.sd));
  memcpy(a.si, w.d.si, sizeof(a.si));
  const int64_t B = w.d.batch;
  const unsigned grid = (unsigned)((B + kSmallThreads - 1) / kSmallThreads);
  const size_t shmem = (size_t)kSmallThreads * w.d.obs_dim * sizeof(float);
  switch (w.d.scenario) {
    case SS_SCN_SIMPLE_SPREAD: {
      // full steps on tile-aligned data go through the bulk-copy pipeline;
      // the (< 128 env) tail and every other mode through the eager kernel
      int64_t ntiles = 0;
      if (pipe_eligible(w, a, NA)) {
        ntiles = B / kPipeTile;
        int rc = SS_OK;
        switch (NA) {
          case 2: rc = launch_pipe<2>(w, a, ntiles, st); break;
          case 3: rc = launch_pipe<3>(w, a, ntiles, st); break;
          case 4: rc = launch_pipe<4>(w, a, ntiles, st); break;
        }
        if (rc) return rc;
      }
      a.e_begin = ntiles * kPipeTile;
      const int64_t rest = B - a.e_begin;
      if (rest <= 0) break;
      const unsigned g2 = (unsigned)((rest + kSmallThreads - 1) / kSmallThreads);
#define SS_CASE(n) case n: launch_step(k_simple_spread<n>, dim3(g2), dim3(kSmallThreads), shmem, st, a); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_TRANSPORT: {
#define SS_CASE(n)                                                                         \
  case n:                                                                                  \
    if (w.d.si[1]) launch_step(k_transport<n, 1>, dim3(grid), dim3(kSmallThreads), shmem, st, a); \
    else launch_step(k_transport<n, 0>, dim3(grid), dim3(kSmallThreads), shmem, st, a);           \
    break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_WHEEL: {
      if (a.mode & SS_DO_PHYSICS) {
        set_error("wheel: physics runs through ss_world_step (generic kernel)");
        return SS_ERR_CONTRACT;
      }
#define SS_CASE(n) case n: launch_step(k_wheel<n>, dim3(grid), dim3(kSmallThreads), shmem, st, a); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_GIVE_WAY: {
      if ((a.mode & SS_DO_PHYSICS) || NA != 2) {
        set_error("give_way: 2 agents; physics runs through ss_world_step (generic kernel)");
        return SS_ERR_CONTRACT;
      }
      launch_step(k_give_way, dim3(grid), dim3(kSmallThreads), shmem, st, a);
      break;
    }
    case SS_SCN_PASSAGE: {
      if (a.mode & SS_DO_PHYSICS) {
        set_error("passage: physics runs through ss_world_step (generic kernel)");
        return SS_ERR_CONTRACT;
      }
#define SS_CASE(n) case n: launch_step(k_passage<n>, dim3(grid), dim3(kSmallThreads), shmem, st, a); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_BALANCE: {
      if (a.mode & SS_DO_PHYSICS) {
        set_error("balance: physics runs through ss_world_step (generic kernel)");
        return SS_ERR_CONTRACT;
      }
#define SS_CASE(n) case n: launch_step(k_balance<n>, dim3(grid), dim3(kSmallThreads), shmem, st, a); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_WATERFALL: {
      if ((a.mode & SS_DO_PHYSICS) || w.d.si[2] > kWaterfallMaxBlocks) {
        set_error("waterfall: at most 8 blocks; physics runs through ss_world_step (generic kernel)");
        return SS_ERR_CONTRACT;
      }
      const size_t wshm = (size_t)kSmallThreads * (w.d.obs_dim | 1) * sizeof(float);
#define SS_CASE(n) case n: launch_step(k_waterfall<n>, dim3(grid), dim3(kSmallThreads), wshm, st, a); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_FOOTBALL: {
      if ((a.mode & SS_DO_PHYSICS) || (NA & 1)) {
        set_error("football: two equal teams; physics runs through ss_world_step (generic kernel)");
        return SS_ERR_CONTRACT;
      }
#define SS_CASE(n) case n: launch_step(k_football<n>, dim3(grid), dim3(kSmallThreads), shmem, st, a); break;
      switch (NA) { SS_CASE(2) SS_CASE(4) SS_CASE(6) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_DROPOUT: {
#define SS_CASE(n) case n: launch_step(k_dropout<n>, dim3(grid), dim3(kSmallThreads), shmem, st, a); break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    case SS_SCN_FLOCKING: {
      if (w.d.si[4] > kFlockMaxRocks) {
        set_error("flocking fused kernel supports at most 6 obstacles");
        return SS_ERR_UNSUPPORTED;
      }
      FlockLidarK lk;
      lk.r2_agent = w.d.sd[0];
      lk.r2_rock = w.d.sd[1];
      lk.agent = make_screen(w.d.sd[2], w.d.lidar_max_range);
      lk.rock = make_screen(w.d.sd[3], w.d.lidar_max_range);
      a.n_rays = w.d.lidar_rays;
      a.lidar_range = w.d.lidar_max_range;
      a.attach_rot = w.d.lidar_attach_rotation;
      a.ray_start = w.d.lidar_start;
      a.ray_span = w.d.lidar_span;
      a.ray_dir = w.d_lidar_dirs;
      if (a.n_rays > 32) {
        set_error("fused flocking lidar supports at most 32 rays");
        return SS_ERR_UNSUPPORTED;
      }
      {
        // uniform fan screen (k_flocking_w): needs 0 < span <= 2 pi
        const double two_pi = 6.283185307179586, span = w.d.lidar_span;
        static const bool no_fan = std::getenv("SS_LIDAR_NO_FAN") != nullptr;
        lk.fan_ok = !no_fan && a.n_rays > 0 && span > 0.0 && span <= two_pi * (1.0 + 1e-12);
        const double step = a.n_rays > 0 ? span / a.n_rays : 1.0;
        lk.fan.start = (float)w.d.lidar_start;
        lk.fan.inv_step = (float)(1.0 / step);
        lk.fan.period = (float)(two_pi / step);
        lk.fan.quarter = (float)(0.25 * two_pi / step);
        lk.fan.n = a.n_rays;
        lk.fan.all = a.n_rays >= 32 ? 0xffffffffu : ((1u << a.n_rays) - 1u);
        lk.fan.full = span == two_pi && lk.fan.period == (float)a.n_rays;
      }
      static const bool legacy = std::getenv("SS_FLOCK_THREAD_PER_ENV") != nullptr;
      if (!legacy) {
        // warp per agent (k_flocking_w): 32 envs per CTA of NA warps
        const size_t wshmem = flocking_w_smem(NA, w.d.si[4], a.n_rays, w.d.obs_dim);
        const unsigned wgrid = (unsigned)((B + 31) / 32);
#define SS_CASE(n)                                                                          \
  case n:                                                                                   \
    if (wshmem > 48 * 1024)                                                                 \
      cudaFuncSetAttribute(k_flocking_w<n>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                           (int)wshmem);                                                    \
    launch_step(k_flocking_w<n>, dim3(wgrid), dim3(32 * n), wshmem, st, a, lk);                                     \
    break;
        switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
        break;
      }
      const size_t fshmem = (size_t)kSmallThreads * (w.d.obs_dim | 1) * sizeof(float) +
                            (size_t)a.n_rays * kSmallThreads * sizeof(double) +
                            (size_t)((a.n_rays + 1) & ~1) * sizeof(float2);
#define SS_CASE(n)                                                                          \
  case n:                                                                                   \
    if (fshmem > 48 * 1024)                                                                 \
      cudaFuncSetAttribute(k_flocking<n>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                           (int)fshmem);                                                    \
    launch_step(k_flocking<n>, dim3(grid), dim3(kSmallThreads), fshmem, st, a, lk);                                \
    break;
      switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
      break;
    }
    default:
      set_error("launch_small: not a small scenario");
      return SS_ERR_SCENARIO;
  }
  return cuda_status(cudaGetLastError(), "fused step launch");
}

}  // namespace ss
