// ss_physics.cuh — world_step (dynamics.py:123-184) for one env of ANY world:
// action / gravity / pair-contact forces and torques over the static pair
// list (closest_points for every sphere / box / line pair), the joint
// extension, then semi-implicit Euler for every movable / rotatable entity,
// repeated for each physics sub-step.  Shared by the generic step kernel
// (k_generic_physics: user scenarios, world_step()) and the fused kernels of
// the line / box catalog tasks, which run it before their reward /
// observation part in the same launch.  State is read from and written to
// global memory (one thread per env, its own rows only); the per-entity
// force / torque accumulators live in shared memory at [k * stride + lane].
#pragma once
#include "ss_geometry.cuh"

namespace ss {

SS_DEV V2 load_pos(const DevState& s, const SsEntityDesc& d, int64_t e) {
  if (d.movable) { const float4 q = s.dyn[d.slot * s.B + e]; return v2(q.x, q.y); }
  const float2 q = s.stat[d.slot * s.B + e];
  return v2(q.x, q.y);
}

// World-frame anchor of a joint end: pos + R(rot) (ox, oy), numpy float32
// cos/sin, separately rounded (the oracle's joint_anchor); a zero offset is
// the position itself.
SS_DEV V2 joint_anchor(const DevState& s, const SsEntityDesc& d, int k, int64_t e, float ox, float oy,
                       V2& pos) {
  pos = load_pos(s, d, e);
  if (ox == 0.0f && oy == 0.0f) return pos;
  const float r = s.rot[k * s.B + e].x;
  const float c = np_cosf(r), sn = np_sinf(r);
  return v2(fadd(pos.x, fsub(fmul(ox, c), fmul(oy, sn))), fadd(pos.y, fadd(fmul(ox, sn), fmul(oy, c))));
}

// Distance-joint penalty force on end a (SsJointDesc, include/swarmsim_b200.h);
// false when the joint exerts no force in this env.
SS_DEV bool joint_force(V2 pa, V2 pb, float target, float stiff, float k, float& fx, float& fy) {
  const float dx = fsub(pa.x, pb.x), dy = fsub(pa.y, pb.y);
  const float dist = fsqrt(fadd(fmul(dx, dx), fmul(dy, dy)));
  if (!(dist >= 1e-6f) || dist == target) return false;
  const bool rep = dist < target;
  const float z = fdiv(rep ? fsub(target, dist) : fsub(dist, target), k);
  const float pen = fmul(np_softplus(z), k);
  const float sf = rep ? stiff : -stiff;
  fx = fmul(fmul(sf, fdiv(dx, dist)), pen);
  fy = fmul(fmul(sf, fdiv(dy, dist)), pen);
  return true;
}

// One Env.step of physics for env e.  agent_force(i, fx, fy) yields agent
// i's force (false: no action, e.g. a missing pointer); it is asked once per
// sub-step and must return the step's held value.  sm holds 3 * E * stride
// floats (FX, FY, TQ).  Returns false on an unsupported shape pair.
template <class AgentForce>
SS_DEV bool env_physics(const DevState& s, const PhysK& ph, const SsEntityDesc* ents,
                        const SsPairDesc* pairs, int E, int P, const SsJointDesc* joints, int J,
                        int A, int64_t e, float* sm, int stride, int lane, AgentForce agent_force) {
  const int64_t B = s.B;
  float* FX = sm;
  float* FY = sm + E * stride;
  float* TQ = sm + 2 * E * stride;
  for (int sub = 0; sub < ph.substeps; ++sub) {
    for (int k = 0; k < E; ++k) {
      FX[k * stride + lane] = 0.0f; FY[k * stride + lane] = 0.0f; TQ[k * stride + lane] = 0.0f;
    }
    for (int i = 0; i < A; ++i) {   // forces[agent] = zeros + action (dynamics.py:151-152)
      float fx, fy;
      if (!agent_force(i, fx, fy)) continue;
      FX[i * stride + lane] = fadd(0.0f, fx);
      FY[i * stride + lane] = fadd(0.0f, fy);
    }
    if (ph.has_gravity) {  // dynamics.py:154-161
      for (int k = 0; k < E; ++k) {
        const SsEntityDesc& d = ents[k];
        if (!d.movable) continue;
        FX[k * stride + lane] = fadd(FX[k * stride + lane], d.grav_x);
        FY[k * stride + lane] = fadd(FY[k * stride + lane], d.grav_y);
      }
    }
    // pair contacts in pair-list order (dynamics.py:163-180)
    for (int p = 0; p < P; ++p) {
      const SsPairDesc pr = pairs[p];
      const SsEntityDesc& di = ents[pr.i];
      const SsEntityDesc& dj = ents[pr.j];
      const V2 pi = load_pos(s, di, e), pj = load_pos(s, dj, e);
      const float ri = s.rot[pr.i * B + e].x, rj = s.rot[pr.j * B + e].x;
      ShapeK si, sj;
      si.kind = di.shape; si.d0 = di.dim0; si.d1 = di.dim1;
      sj.kind = dj.shape; sj.d0 = dj.dim0; sj.d1 = dj.dim1;
      V2 oi, oj;
      if (!closest_points(pi, ri, si, pj, rj, sj, oi, oj)) return false;
      float fx, fy;
      if (!contact_force(oi.x, oi.y, oj.x, oj.y, pr.d_min, pr.d2_act, pr.sign, ph.ck, ph.k, fx, fy)) continue;
      FX[pr.i * stride + lane] = fadd(FX[pr.i * stride + lane], fx);
      FY[pr.i * stride + lane] = fadd(FY[pr.i * stride + lane], fy);
      FX[pr.j * stride + lane] = fsub(FX[pr.j * stride + lane], fx);
      FY[pr.j * stride + lane] = fsub(FY[pr.j * stride + lane], fy);
      if (di.rotatable) {
        const V2 r = vsub(oi, pi);
        TQ[pr.i * stride + lane] = fadd(TQ[pr.i * stride + lane], fsub(fmul(r.x, fy), fmul(r.y, fx)));
      }
      if (dj.rotatable) {
        const V2 r = vsub(oj, pj);
        TQ[pr.j * stride + lane] = fsub(TQ[pr.j * stride + lane], fsub(fmul(r.x, fy), fmul(r.y, fx)));
      }
    }
    // joint constraints (extension, SsJointDesc), joint-list order
    for (int q = 0; q < J; ++q) {
      const SsJointDesc jt = joints[q];
      const SsEntityDesc& da = ents[jt.a];
      const SsEntityDesc& db = ents[jt.b];
      V2 pa, pb;
      const V2 qa = joint_anchor(s, da, jt.a, e, jt.ox_a, jt.oy_a, pa);
      const V2 qb = joint_anchor(s, db, jt.b, e, jt.ox_b, jt.oy_b, pb);
      float fx, fy;
      if (!joint_force(qa, qb, jt.dist, jt.stiffness, ph.k, fx, fy)) continue;
      FX[jt.a * stride + lane] = fadd(FX[jt.a * stride + lane], fx);
      FY[jt.a * stride + lane] = fadd(FY[jt.a * stride + lane], fy);
      FX[jt.b * stride + lane] = fsub(FX[jt.b * stride + lane], fx);
      FY[jt.b * stride + lane] = fsub(FY[jt.b * stride + lane], fy);
      if (da.rotatable && jt.rotate_a) {
        const V2 r = vsub(qa, pa);
        TQ[jt.a * stride + lane] = fadd(TQ[jt.a * stride + lane], fsub(fmul(r.x, fy), fmul(r.y, fx)));
      }
      if (db.rotatable && jt.rotate_b) {
        const V2 r = vsub(qb, pb);
        TQ[jt.b * stride + lane] = fsub(TQ[jt.b * stride + lane], fsub(fmul(r.x, fy), fmul(r.y, fx)));
      }
    }
    // integrate (dynamics.py:182-184)
    for (int k = 0; k < E; ++k) {
      const SsEntityDesc& d = ents[k];
      if (d.movable) {
        float4 q = s.dyn[d.slot * B + e];
        integrate_lin(q.x, q.y, q.z, q.w, FX[k * stride + lane], FY[k * stride + lane], ph.keep,
                      d.inv_m_dt, ph.dt, d.max_speed);
        s.dyn[d.slot * B + e] = q;
      }
      if (d.rotatable) {
        float2 r = s.rot[k * B + e];
        integrate_ang(r.x, r.y, TQ[k * stride + lane], ph.keep, d.inv_i_dt, ph.dt);
        s.rot[k * B + e] = r;
      }
    }
  }
  return true;
}

}  // namespace ss
