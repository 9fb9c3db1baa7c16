// ss_geometry.cuh — closest points between posed shapes (geometry.py:21-163),
// restated per env with numpy's float32/float64 rounding.  Sphere support is
// its centre, boxes are hollow perimeters, lines are segments.
#pragma once
#include "ss_internal.cuh"

namespace ss {

struct V2 { float x, y; };

SS_DEV V2 v2(float x, float y) { V2 r; r.x = x; r.y = y; return r; }
SS_DEV V2 vsub(V2 a, V2 b) { return v2(fsub(a.x, b.x), fsub(a.y, b.y)); }
SS_DEV V2 vadd(V2 a, V2 b) { return v2(fadd(a.x, b.x), fadd(a.y, b.y)); }
SS_DEV V2 vmul(V2 a, float s) { return v2(fmul(a.x, s), fmul(a.y, s)); }
SS_DEV float vdot(V2 a, V2 b) { return fadd(fmul(a.x, b.x), fmul(a.y, b.y)); }
SS_DEV float clip01(float t) { return fminf(fmaxf(t, 0.0f), 1.0f); }

// np.cos / np.sin of a float32 angle, bit-exact (ss_math.cuh np_sincosf).
SS_DEV void cos_sin(float rot, float& ca, float& sa) {
  if (rot == 0.0f) { ca = 1.0f; sa = rot; return; }
  ca = np_cosf(rot);
  sa = np_sinf(rot);
}

// segment_endpoints (geometry.py:21-26); half is a Python double.
SS_DEV void segment_endpoints(V2 pos, float rot, double length, V2& a, V2& b) {
  const float half = (float)(length / 2);
  float ca, sa; cos_sin(rot, ca, sa);
  const V2 off = v2(fmul(ca, half), fmul(sa, half));
  a = vsub(pos, off);
  b = vadd(pos, off);
}

// box_corners (geometry.py:29-37), counter-clockwise from (+l/2, +w/2).
SS_DEV void box_corners(V2 pos, float rot, double length, double width, V2 c[4]) {
  const float hx = (float)(length / 2), hy = (float)(width / 2);
  float ca, sa; cos_sin(rot, ca, sa);
  const float lx[4] = {hx, -hx, -hx, hx};
  const float ly[4] = {hy, hy, -hy, -hy};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c[k].x = fsub(fadd(pos.x, fmul(lx[k], ca)), fmul(ly[k], sa));
    c[k].y = fadd(fadd(pos.y, fmul(lx[k], sa)), fmul(ly[k], ca));
  }
}

// closest_point_on_segment (geometry.py:44-48).
SS_DEV V2 closest_on_segment(V2 p, V2 a, V2 b) {
  const V2 ab = vsub(b, a);
  const float denom = vdot(ab, ab);
  const float t = clip01(fdiv(vdot(vsub(p, a), ab), fmaxf(denom, 1e-12f)));
  return vadd(a, vmul(ab, t));
}

// closest_points_segment_segment (geometry.py:51-76).
SS_DEV void closest_seg_seg(V2 p1, V2 q1, V2 p2, V2 q2, V2& o1, V2& o2) {
  const V2 d1 = vsub(q1, p1), d2 = vsub(q2, p2), r = vsub(p1, p2);
  const float a = vdot(d1, d1), e = vdot(d2, d2), b = vdot(d1, d2);
  const float c = vdot(d1, r), f = vdot(d2, r);
  const float denom = fsub(fmul(a, e), fmul(b, b));
  const bool nondeg = denom > 1e-12f;
  float s = nondeg ? clip01(fdiv(fsub(fmul(b, f), fmul(c, e)), denom)) : 0.0f;
  const float t = fdiv(fadd(fmul(b, s), f), fmaxf(e, 1e-12f));
  const float t_cl = clip01(t);
  if (t != t_cl) s = clip01(fdiv(fsub(fmul(b, t_cl), c), fmaxf(a, 1e-12f)));
  o1 = vadd(p1, vmul(d1, s));
  o2 = vadd(p2, vmul(d2, t_cl));
}

struct ShapeK {
  int kind;       // SsShape
  double d0, d1;  // python doubles: radius | length,width | length
};

// closest_points (geometry.py:120-156) for shapes in canonical order.
SS_DEV bool closest_points_canon(V2 pi, float ri, const ShapeK& si, V2 pj, float rj,
                                 const ShapeK& sj, V2& oi, V2& oj) {
  if (si.kind == SS_SPHERE && sj.kind == SS_SPHERE) { oi = pi; oj = pj; return true; }
  if (si.kind == SS_SPHERE && sj.kind == SS_LINE) {
    V2 a, b; segment_endpoints(pj, rj, sj.d0, a, b);
    oi = pi; oj = closest_on_segment(pi, a, b); return true;
  }
  if (si.kind == SS_SPHERE && sj.kind == SS_BOX) {
    float ca, sa; cos_sin(rj, ca, sa);
    oi = pi;
    closest_point_on_box(pi.x, pi.y, pj.x, pj.y, ca, sa, sj.d0 / 2, sj.d1 / 2, oj.x, oj.y);
    return true;
  }
  if (si.kind == SS_LINE && sj.kind == SS_LINE) {
    V2 a1, b1, a2, b2;
    segment_endpoints(pi, ri, si.d0, a1, b1);
    segment_endpoints(pj, rj, sj.d0, a2, b2);
    closest_seg_seg(a1, b1, a2, b2, oi, oj); return true;
  }
  if (si.kind == SS_LINE && sj.kind == SS_BOX) {
    V2 a, b, c[4];
    segment_endpoints(pi, ri, si.d0, a, b);
    box_corners(pj, rj, sj.d0, sj.d1, c);
    float best = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      V2 u, v; closest_seg_seg(a, b, c[k], c[(k + 1) & 3], u, v);
      const V2 d = vsub(u, v);
      const float d2 = vdot(d, d);
      if (k == 0 || d2 < best) { best = d2; oi = u; oj = v; }   // argmin: first min wins
    }
    return true;
  }
  if (si.kind == SS_BOX && sj.kind == SS_BOX) {
    V2 ci[4], cj[4];
    box_corners(pi, ri, si.d0, si.d1, ci);
    box_corners(pj, rj, sj.d0, sj.d1, cj);
    float best = 0.0f;
    bool first = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        V2 u, v; closest_seg_seg(ci[k], ci[(k + 1) & 3], cj[l], cj[(l + 1) & 3], u, v);
        const V2 d = vsub(u, v);
        const float d2 = vdot(d, d);
        if (first || d2 < best) { best = d2; oi = u; oj = v; first = false; }
      }
    }
    return true;
  }
  return false;
}

// closest_points (geometry.py:120-163): canonical order, else the mirrored
// order (geometry.py:157-162); false for an unsupported pair.
SS_DEV bool closest_points(V2 pi, float ri, const ShapeK& si, V2 pj, float rj, const ShapeK& sj,
                           V2& oi, V2& oj) {
  if (((si.kind == SS_LINE || si.kind == SS_BOX) && sj.kind == SS_SPHERE) ||
      (si.kind == SS_BOX && sj.kind == SS_LINE)) {
    return closest_points_canon(pj, rj, sj, pi, ri, si, oj, oi);
  }
  return closest_points_canon(pi, ri, si, pj, rj, sj, oi, oj);
}

}  // namespace ss
