// ss_lidar.cu — lidar_scan (sensors.py:113-146) for any world: fp64 ray casts
// against every collidable entity except the emitter, nearest hit capped at
// max_range and cast to float32.  One thread per (env, ray); out[e][m] is
// written coalesced.
#include "ss_geometry.cuh"

namespace ss {

SS_DEV double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// sensors.py:43-54
SS_DEV double ray_circle_d(double ox, double oy, double dx, double dy, double cx, double cy,
                           double r2) {
  const double fx = dsub_rn(ox, cx), fy = dsub_rn(oy, cy);
  const double b = dadd_rn(dmul_rn(fx, dx), dmul_rn(fy, dy));
  const double c = dsub_rn(dadd_rn(dmul_rn(fx, fx), dmul_rn(fy, fy)), r2);
  const double disc = dsub_rn(dmul_rn(b, b), c);
  if (!(disc >= 0.0)) return dinf();
  const double sq = sqrt(disc);
  const double t1 = dsub_rn(-b, sq), t2 = dadd_rn(-b, sq);
  if (t1 > 1e-9) return t1;
  if (t2 > 1e-9) return t2;
  return dinf();
}

// sensors.py:57-66
SS_DEV double ray_segment_d(double ox, double oy, double dx, double dy, double ax, double ay,
                            double bx, double by) {
  const double ex = dsub_rn(bx, ax), ey = dsub_rn(by, ay);
  const double denom = dsub_rn(dmul_rn(dx, ey), dmul_rn(dy, ex));
  if (!(fabs(denom) >= 1e-12)) return dinf();
  const double qx = dsub_rn(ax, ox), qy = dsub_rn(ay, oy);
  const double t = dsub_rn(dmul_rn(qx, ey), dmul_rn(qy, ex)) / denom;
  const double u = dsub_rn(dmul_rn(qx, dy), dmul_rn(qy, dx)) / denom;
  if (t > 1e-9 && u >= 0.0 && u <= 1.0) return t;
  return dinf();
}

// sensors.py:69-92 (slab test in the box frame)
SS_DEV double ray_rect_d(double ox, double oy, double dx, double dy, double cx, double cy,
                         double rot, double hx, double hy) {
  double sa, ca;
  sincos(rot, &sa, &ca);
  const double rx = dsub_rn(ox, cx), ry = dsub_rn(oy, cy);
  const double lo[2] = {dadd_rn(dmul_rn(rx, ca), dmul_rn(ry, sa)), dadd_rn(dmul_rn(-rx, sa), dmul_rn(ry, ca))};
  const double ld[2] = {dadd_rn(dmul_rn(dx, ca), dmul_rn(dy, sa)), dadd_rn(dmul_rn(-dx, sa), dmul_rn(dy, ca))};
  const double hh[2] = {hx, hy};
  double tmin = -dinf(), tmax = dinf();
  bool miss = false;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool par = fabs(ld[k]) < 1e-12;
    if (par) {
      miss |= fabs(lo[k]) > hh[k];
    } else {
      const double t_lo = dsub_rn(-hh[k], lo[k]) / ld[k];
      const double t_hi = dsub_rn(hh[k], lo[k]) / ld[k];
      tmin = fmax(tmin, fmin(t_lo, t_hi));
      tmax = fmin(tmax, fmax(t_lo, t_hi));
    }
  }
  const bool hit = !miss && (tmax >= fmax(tmin, 1e-9));
  if (!hit) return dinf();
  return tmin > 1e-9 ? tmin : tmax;
}

// Nearest hit over the collidable entities except `skip` (sensors.py:95-135):
// ties resolve to the smallest t (min is order independent).
SS_DEV double nearest_hit(const DevState& s, const SsEntityDesc* ents, int E, int skip, int64_t e,
                          float px, float py, double dx, double dy) {
  const int64_t B = s.B;
  const double ox = px, oy = py;
  double best = dinf();
  for (int k = 0; k < E; ++k) {
    const SsEntityDesc& d = ents[k];
    if (!d.collidable || k == skip) continue;
    double cx, cy;
    if (d.movable) { const float4 q = s.dyn[d.slot * B + e]; cx = q.x; cy = q.y; }
    else { const float2 q = s.stat[d.slot * B + e]; cx = q.x; cy = q.y; }
    double t;
    if (d.shape == SS_SPHERE) {
      t = ray_circle_d(ox, oy, dx, dy, cx, cy, dmul_rn(d.dim0, d.dim0));
    } else if (d.shape == SS_LINE) {
      const double r = (double)s.rot[k * B + e].x;
      const double half = d.dim0 / 2;
      double sr, cr;
      sincos(r, &sr, &cr);
      const double ex = dmul_rn(cr, half), ey = dmul_rn(sr, half);
      t = ray_segment_d(ox, oy, dx, dy, dsub_rn(cx, ex), dsub_rn(cy, ey), dadd_rn(cx, ex),
                        dadd_rn(cy, ey));
    } else {
      t = ray_rect_d(ox, oy, dx, dy, cx, cy, (double)s.rot[k * B + e].x, d.dim0 / 2, d.dim1 / 2);
    }
    best = fmin(best, t);
  }
  return best;
}

struct LidarArgs {
  DevState s;
  const SsEntityDesc* ents;
  int E;
  int emitter;
  int n_rays;
  double max_range, start, span;
  int attach_rot;
  const double* dirs;   // optional [n_rays][2] for rot == 0
  float* out;
};

__global__ void __launch_bounds__(256) k_lidar(const LidarArgs a) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t B = a.s.B;
  if (idx >= B * a.n_rays) return;
  const int64_t e = idx / a.n_rays;
  const int m = (int)(idx - e * a.n_rays);
  const SsEntityDesc& me = a.ents[a.emitter];
  float px, py;
  if (me.movable) { const float4 q = a.s.dyn[me.slot * B + e]; px = q.x; py = q.y; }
  else { const float2 q = a.s.stat[me.slot * B + e]; px = q.x; py = q.y; }
  const float rot = a.attach_rot ? a.s.rot[a.emitter * B + e].x : 0.0f;
  double dx, dy;
  if (rot == 0.0f && a.dirs) { dx = a.dirs[2 * m]; dy = a.dirs[2 * m + 1]; }
  else {
    const double ang = dadd_rn(dadd_rn(a.start, (double)m * a.span / a.n_rays), (double)rot);
    sincos(ang, &dy, &dx);
  }
  a.out[e * a.n_rays + m] =
      (float)fmin(nearest_hit(a.s, a.ents, a.E, a.emitter, e, px, py, dx, dy), a.max_range);
}

// cast_ray (sensors.py:113-135): one ray per env from an arbitrary origin.
__global__ void __launch_bounds__(256) k_cast_ray(DevState s, const SsEntityDesc* ents, int E,
                                                  int exclude, const float* ox, const float* oy,
                                                  const double* angle, double max_range,
                                                  float* out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= s.B) return;
  double dx, dy;
  sincos(angle[e], &dy, &dx);
  out[e] = (float)fmin(nearest_hit(s, ents, E, exclude, e, ox[e], oy[e], dx, dy), max_range);
}

int launch_lidar(World& w, const SsBuffers* buf, int agent, const SsLidarDesc* lidar, float* out,
                 cudaStream_t st) {
  LidarArgs a;
  memset(&a, 0, sizeof(a));
  a.s = make_state(w, buf);
  a.ents = w.d_ents;
  a.E = w.d.n_entities;
  a.emitter = agent;
  a.n_rays = lidar->n_rays;
  a.max_range = lidar->max_range;
  a.start = lidar->start_angle;
  a.span = lidar->span;
  a.attach_rot = lidar->attach_rotation;
  a.dirs = lidar->dir_table;
  a.out = out;
  const int64_t n = w.d.batch * lidar->n_rays;
  k_lidar<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "lidar launch");
}

int launch_cast_ray(World& w, const SsBuffers* buf, int exclude, const float* ox, const float* oy,
                    const double* angle, double max_range, float* out, cudaStream_t st) {
  const DevState s = make_state(w, buf);
  const int64_t n = w.d.batch;
  k_cast_ray<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s, w.d_ents, w.d.n_entities, exclude, ox,
                                                          oy, angle, max_range, out);
  return cuda_status(cudaGetLastError(), "cast_ray launch");
}

}  // namespace ss
