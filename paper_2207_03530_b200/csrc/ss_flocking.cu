// ss_flocking.cu — fused Env.step of flocking with the Lidar extension
// (scenarios/flocking.py + sensors.py): k_flocking_w (warp per agent) and the
// legacy thread-per-env k_flocking.
#include "ss_small.cuh"

namespace ss {

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

constexpr int kLidarQueue = 128;   // (lane, target, ray) tests staged per warp and round

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
#ifndef SS_LIDAR_ROLLED
#define SS_LIDAR_ROLLED 0
#endif
template <int NA>
SS_DEV void lidar_fan_warp(bool active, int i, int lane, int NO, float mex, float mey,
                           const float2* spos, const float2* sst, const FlockLidarK& lk,
                           const double2* sdird, uint32_t* best, int P, uint32_t* queue, int n_rays,
                           uint32_t init_bits) {
  constexpr int NT = NA - 1 + kFlockMaxRocks;
  uint32_t mk[NT];
  int cnt = 0;
  // SS_LIDAR_ROLLED: the per-target loops rolled (one copy of the screen
  // code; the masks then live in local memory) to shrink the hot code
#if SS_LIDAR_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
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
  // minima start at float(max_range): min(float(R), float(t)...) ==
  // float(min(R, t...)) (rounding is monotone), so the cap is folded in
  for (int m = 0; m < n_rays; ++m) best[lane * P + m] = init_bits;
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
#if SS_LIDAR_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
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
// Cold lidar paths of k_flocking_w, out of line (the fan screen is the hot
// one): the per-ray screen when the fan is not uniform, and attached
// rotations (sensors.py:121-135: per-ray fp64 angles).
#ifndef SS_FLOCK_CONTACT
#define SS_FLOCK_CONTACT contact_force_ol   // contact_force: inline at every call site
#endif
template <int NA>
__device__ __noinline__ void flock_lidar_screened(int i, int lane, int NO, float4 me, const float2* spos,
                                                  const float2* sst, const float2* sdir, const double2* sdird,
                                                  RayScreen s_agent, RayScreen s_rock, double r2_agent,
                                                  double r2_rock, int n_rays, float range_f, uint32_t* best) {
  const double ox = (double)me.x, oy = (double)me.y;
  for (int m = 0; m < n_rays; ++m) best[m] = 0x7f800000u;
  for (int o = 0; o < NA; ++o) {
    if (o == i) continue;
    const float2 q = spos[o * 32 + lane];
    const uint32_t mk = ray_mask(me.x - q.x, me.y - q.y, sdir, n_rays, s_agent);
    ray_hits_f(mk, ox, oy, sdird, (double)q.x, (double)q.y, r2_agent, best, 1);
  }
  for (int r = 0; r < NO; ++r) {
    const float2 q = sst[(1 + r) * 32 + lane];
    const uint32_t mk = ray_mask(me.x - q.x, me.y - q.y, sdir, n_rays, s_rock);
    ray_hits_f(mk, ox, oy, sdird, (double)q.x, (double)q.y, r2_rock, best, 1);
  }
  for (int m = 0; m < n_rays; ++m) best[m] = __float_as_uint(fminf(__uint_as_float(best[m]), range_f));
}

template <int NA>
__device__ __noinline__ void flock_lidar_rotated(int i, int lane, int NO, float4 me, float rot_i,
                                                 const float2* spos, const float2* sst, double r2_agent,
                                                 double r2_rock, int n_rays, double ray_start, double ray_span,
                                                 double lidar_range, float* out) {
  const double ox = (double)me.x, oy = (double)me.y;
  for (int m = 0; m < n_rays; ++m) {
    const double ang = dadd_rn(dadd_rn(ray_start, (double)m * ray_span / n_rays), (double)rot_i);
    double dx, dy;
    sincos(ang, &dy, &dx);
    double b = __longlong_as_double(0x7ff0000000000000LL);
    for (int o = 0; o < NA; ++o) {
      if (o == i) continue;
      const float2 q = spos[o * 32 + lane];
      b = fmin(b, ray_circle(ox, oy, dx, dy, (double)q.x, (double)q.y, r2_agent));
    }
    for (int r = 0; r < NO; ++r) {
      const float2 q = sst[(1 + r) * 32 + lane];
      b = fmin(b, ray_circle(ox, oy, dx, dy, (double)q.x, (double)q.y, r2_rock));
    }
    out[m] = (float)fmin(b, lidar_range);
  }
}

// ROLL: the fused rollout (RolloutArgs *ro, SS_MODE_STEP): the steps of
// the replay in one launch, the agents' rows kept in registers and the
// beacon / rocks staged once; the per-step pointers come from ro.
template <int NA, bool ROLL>
SS_DEV void flocking_w_body(const SmallArgs& a, const FlockLidarK& lk, const RolloutArgs* ro) {
  extern __shared__ __align__(16) float smem_w[];
  const int NO = a.si[4];
  const int O = a.obs_dim;
  const int P = O | 1;
  const int lane = threadIdx.x & 31, i = threadIdx.x >> 5;
  const int64_t B = a.s.B;
  const int64_t e0 = (int64_t)blockIdx.x * 32;
  const int64_t e = e0 + lane;
  const bool valid = e < B;
  const int nvalid = (int)min((int64_t)32, B - e0);
  // shared memory: [dirs: n_rays double2][agents: NA x 32 float2 post-step positions]
  //                [queue: NA x kLidarQueue u32][dirs: n_rays(+1) float2]
  //                [static: (1+NO) x 32 float2][rows: NA warps x 32 x P]
  // The pre-step agent copy (NA x 32 float4, read only by the physics)
  // aliases the start of the rows region, which is first written after the
  // barrier that ends the physics.  (pre / post copies: one barrier between
  // physics and the rest; the lidar minima live in the rows' lidar columns)
  double2* sdird = reinterpret_cast<double2*>(smem_w);
  float2* spos = reinterpret_cast<float2*>(sdird + a.n_rays);
  uint32_t* squeue = reinterpret_cast<uint32_t*>(spos + NA * 32);
  float2* sdir = reinterpret_cast<float2*>(squeue + NA * kLidarQueue);
  float2* sst = reinterpret_cast<float2*>(sdir + ((a.n_rays + 1) & ~1));
  float* rows = reinterpret_cast<float*>(sst + (1 + NO) * 32);
  float4* sag = reinterpret_cast<float4*>(rows);
  float* srow = rows + i * 32 * P;
  if (threadIdx.x < a.n_rays) {
    const double dx = a.ray_dir[2 * threadIdx.x], dy = a.ray_dir[2 * threadIdx.x + 1];
    sdird[threadIdx.x] = make_double2(dx, dy);
    sdir[threadIdx.x] = make_float2((float)dx, (float)dy);
  }
  float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t steps = 0;
  const int mode = ROLL ? SS_MODE_STEP : a.mode;
  if (valid) {
    // every global load of the step issued up front
    me = a.s.dyn[i * B + e];
    if (mode & (SS_DO_COUNT | SS_DO_DONE)) steps = a.s.step_count[e];
    for (int k = i; k < 1 + NO; k += NA) sst[k * 32 + lane] = a.s.stat[k * B + e];
  }
  const int n_steps = ROLL ? rollout_len(ro->guard, ro->n_steps) : 1;
  for (int step = 0; step < n_steps; ++step) {
  const float2* act_i = ROLL ? ro->act[step][i] : a.act[i];
  float* const obs_out = ROLL ? ro->obs[step] : a.obs;
  float* const rew_out = ROLL ? ro->rew[step] : a.rew;
  uint8_t* const done_out = ROLL ? ro->done[step] : a.done;
  float2 u = make_float2(0.f, 0.f);
  if (valid && (mode & SS_DO_PHYSICS)) u = act_i[e];
  // (rollout) every warp is done with the previous step's rows, positions
  // and lidar queue before the pre-step copy overwrites the rows region
  if (ROLL && step > 0) __syncthreads();
  if (valid) sag[i * 32 + lane] = me;
  __syncthreads();
  if (mode & SS_DO_PHYSICS) {
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
        if (SS_FLOCK_CONTACT(q.x, q.y, me.x, me.y, dmin_aa, d2_aa, sign, a.ph.ck, a.ph.k, cx, cy)) {
          fx = fsub(fx, cx); fy = fsub(fy, cy);
        }
      } else {
        if (SS_FLOCK_CONTACT(me.x, me.y, q.x, q.y, dmin_aa, d2_aa, sign, a.ph.ck, a.ph.k, cx, cy)) {
          fx = fadd(fx, cx); fy = fadd(fy, cy);
        }
      }
    }
    for (int r = 0; r < NO; ++r) {
      const float2 q = sst[(1 + r) * 32 + lane];
      const float sign = ((i + NA + 1 + r) & 1) ? -1.0f : 1.0f;
      float cx, cy;
      if (SS_FLOCK_CONTACT(me.x, me.y, q.x, q.y, dmin_ar, d2_ar, sign, a.ph.ck, a.ph.k, cx, cy)) {
        fx = fadd(fx, cx); fy = fadd(fy, cy);
      }
    }
    integrate_lin(me.x, me.y, me.z, me.w, fx, fy, a.ph.keep, d.inv_m_dt, a.ph.dt, d.max_speed);
    }
    }
    if (valid && !ROLL) a.s.dyn[i * B + e] = me;
  }
  if (valid) spos[i * 32 + lane] = make_float2(me.x, me.y);
  __syncthreads();                       // post-step positions of every agent staged
  if (valid && (mode & SS_DO_COUNT)) { steps += 1; if (i == 0 && !ROLL) a.s.step_count[e] = steps; }
  const float2 beacon = valid ? sst[lane] : make_float2(0.f, 0.f);
  if (valid && (mode & SS_DO_REWARD)) {
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
    __stcs(rew_out + i * B + e, fsub(-gap, fmul(pen, fadd(ca, cr))));
  }
  if (valid && i == 0 && (mode & SS_DO_DONE)) done_out[e] = (uint8_t)(steps >= a.ph.max_steps);
  if (mode & SS_DO_OBS) {
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
      const float rot_i = (valid && a.attach_rot) ? a.s.rot[i * B + e].x : 0.0f;
      const bool fan = valid && rot_i == 0.0f;
      uint32_t* wbest = reinterpret_cast<uint32_t*>(srow + c);   // this warp's rows, lidar columns
      uint32_t* best = wbest + lane * P;
      const float range_f = (float)a.lidar_range;
      if (lk.fan_ok) {
        // warp-collective: all lanes, including invalid / rotated ones
        lidar_fan_warp<NA>(fan, i, lane, NO, me.x, me.y, spos, sst, lk, sdird, wbest, P, squeue + i * kLidarQueue,
                           a.n_rays, __float_as_uint(range_f));
      } else if (fan) {
        flock_lidar_screened<NA>(i, lane, NO, me, spos, sst, sdir, sdird, lk.agent, lk.rock, lk.r2_agent,
                                 lk.r2_rock, a.n_rays, range_f, best);
      }
      if (valid && !fan)
        flock_lidar_rotated<NA>(i, lane, NO, me, rot_i, spos, sst, lk.r2_agent, lk.r2_rock, a.n_rays,
                                a.ray_start, a.ray_span, a.lidar_range, row + c);
    }
    if (nvalid > 0) warp_flush_padded(obs_out + i * a.obs_stride + e0 * O, nvalid, O, P, srow);
  }
  }   // steps
  if (ROLL && valid) {
    a.s.dyn[i * B + e] = me;
    if (i == 0) a.s.step_count[e] = steps;
  }
}

template <int NA>
__global__ void __launch_bounds__(32 * NA, (SS_FLOCK_WARPS / NA < 32 ? SS_FLOCK_WARPS / NA : 32))
    k_flocking_w(const SmallArgs a, const FlockLidarK lk) {
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  flocking_w_body<NA, false>(a, lk, nullptr);
}

// flocking, fused open-loop rollout (SsRolloutIO): ro.n_steps steps of
// k_flocking_w's work per launch, each env's agents kept on chip between them.
template <int NA>
__global__ void __launch_bounds__(32 * NA, (SS_FLOCK_WARPS / NA < 32 ? SS_FLOCK_WARPS / NA : 32))
    k_flocking_w_rollout(const RolloutArgs ro, const FlockLidarK lk) {
  grid_dep_sync();
  flocking_w_body<NA, true>(ro.a, lk, &ro);
}

inline size_t flocking_w_smem(int NA, int NO, int n_rays, int O) {
  const size_t rows = (size_t)NA * 32 * (O | 1) * sizeof(float), pre = (size_t)NA * 32 * sizeof(float4);
  return (size_t)n_rays * sizeof(double2) + (size_t)NA * 32 * sizeof(float2) +
         (size_t)NA * kLidarQueue * sizeof(uint32_t) + (size_t)((n_rays + 1) & ~1) * sizeof(float2) +
         (size_t)(1 + NO) * 32 * sizeof(float2) + (rows > pre ? rows : pre);
}

// Lidar constants of a flocking launch (a's lidar fields, the screens and
// the uniform fan); SS_OK or an error status.
static int flock_setup(World& w, SmallArgs& a, FlockLidarK& lk) {
  if (w.d.si[4] > kFlockMaxRocks) {
    set_error("flocking fused kernel supports at most 6 obstacles");
    return SS_ERR_UNSUPPORTED;
  }
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
  return SS_OK;
}

static bool flock_legacy() {
  static const bool legacy = std::getenv("SS_FLOCK_THREAD_PER_ENV") != nullptr;
  return legacy;
}

int launch_flocking_rollout(World& w, RolloutArgs& r, cudaStream_t st) {
  FlockLidarK lk;
  const int rc = flock_setup(w, r.a, lk);
  if (rc != SS_OK) return rc;
  if (flock_legacy()) { set_error("no flocking rollout on the thread-per-env kernel"); return SS_ERR_UNSUPPORTED; }
  const int NA = w.d.n_agents;
  const size_t wshmem = flocking_w_smem(NA, w.d.si[4], r.a.n_rays, w.d.obs_dim);
  const unsigned wgrid = (unsigned)((w.d.batch + 31) / 32);
#define SS_CASE(n)                                                                                        \
  case n:                                                                                                 \
    if (wshmem > 48 * 1024)                                                                               \
      cudaFuncSetAttribute(k_flocking_w_rollout<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wshmem); \
    launch_step(k_flocking_w_rollout<n>, dim3(wgrid), dim3(32 * n), wshmem, st, r, lk);                  \
    break;
  switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
  return cuda_status(cudaGetLastError(), "flocking rollout launch");
}

int launch_flocking(World& w, SmallArgs& a, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const int64_t B = w.d.batch;
  const unsigned grid = (unsigned)((B + kSmallThreads - 1) / kSmallThreads);
  FlockLidarK lk;
  {
    const int rc = flock_setup(w, a, lk);
    if (rc != SS_OK) return rc;
  }
  if (!flock_legacy()) {
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
    return cuda_status(cudaGetLastError(), "flocking step launch");
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
  return cuda_status(cudaGetLastError(), "flocking step launch");
}

}  // namespace ss
