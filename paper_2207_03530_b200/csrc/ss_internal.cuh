// ss_internal.cuh — library-private world descriptor and device helpers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/swarmsim_b200.h"
#include "ss_math.cuh"

namespace ss {

using namespace ssm;

// Library-owned copy of the SsWorldDesc plus device mirrors of its tables.
struct World {
  SsWorldDesc d;                       // scalars (pointers below replace d's)
  std::vector<SsEntityDesc> ents;
  std::vector<SsPairDesc> pairs;
  std::vector<SsResetOp> reset_ops;
  std::vector<SsJointDesc> joints;
  SsEntityDesc* d_ents = nullptr;      // device copies
  SsJointDesc* d_joints = nullptr;
  SsPairDesc* d_pairs = nullptr;
  SsResetOp* d_reset_ops = nullptr;
  double* d_lidar_dirs = nullptr;      // [lidar_rays][2]
  int64_t* d_scan = nullptr;           // masked-reset block scan scratch
  int64_t scan_cap = 0;
  int n_slots = 0;                     // draw slots per env of the reset program
};

void set_error(const std::string& msg);
int cuda_status(cudaError_t e, const char* what);

// Kernel-side view of the state buffers for one call.
struct DevState {
  int64_t B;
  int64_t env_offset;
  int64_t global_batch;
  float4* dyn;        // [n_dyn][B]
  float2* stat;       // [n_stat][B]
  float2* stat_vel;   // [n_stat][B]
  float2* rot;        // [n_entities][B]
  int64_t* step_count;
  uint32_t* flags;
  float* aux;
  const uint64_t* rng_in;
  uint64_t* rng_out;
};

inline DevState make_state(const World& w, const SsBuffers* b) {
  DevState s;
  s.B = w.d.batch;
  s.env_offset = w.d.env_offset;
  s.global_batch = w.d.global_batch;
  s.dyn = reinterpret_cast<float4*>(b->dyn);
  s.stat = reinterpret_cast<float2*>(b->stat);
  s.stat_vel = reinterpret_cast<float2*>(b->stat_vel);
  s.rot = reinterpret_cast<float2*>(b->rot);
  s.step_count = b->step_count;
  s.flags = b->flags;
  s.aux = b->aux;
  s.rng_in = b->rng + (b->rng_cur ? SS_RNG_WORDS : 0);
  s.rng_out = b->rng + (b->rng_cur ? 0 : SS_RNG_WORDS);
  return s;
}

// Physics constants shared by every step kernel.
struct PhysK {
  float dt, keep, ck, k;   // dt: the SUB-step f32(dt / substeps)
  int has_gravity;
  int substeps;            // physics sub-steps per Env.step (1 = reference)
  int64_t max_steps;
};

inline PhysK make_phys(const World& w) {
  PhysK p;
  p.dt = w.d.dt; p.keep = w.d.keep; p.ck = w.d.contact_ck; p.k = w.d.contact_k;
  p.has_gravity = w.d.has_gravity; p.max_steps = w.d.max_steps;
  p.substeps = w.d.substeps > 0 ? w.d.substeps : 1;
  return p;
}

// ---------------------------------------------------------------------------
// Device physics helpers (bit-faithful restatements, numerics in ss_math.cuh)
// ---------------------------------------------------------------------------
#define SS_DEV __device__ __forceinline__

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Step kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (launch_step), so the
// next step's grid is launched while this one drains instead of after it.
// Every such kernel starts with grid_dep_sync(): it waits until the previous
// grid in the stream has completed with its memory visible (no data is
// touched before), then releases its own dependents — they can only launch
// once all of this grid's CTAs are resident, so they never take a slot this
// grid still needs.  Without the attribute both instructions are no-ops.
// ---------------------------------------------------------------------------
SS_DEV void grid_dep_sync() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();   // SS_NO_PDL unset

// The NaN verdict (SsStepIO.guard): the launch is a no-op when any of its n
// guard words is set — word k is step k's action scan inside a multi-step
// graph, so step k stops on a NaN in any action set up to its own.
SS_DEV bool guard_tripped(const int* g, int n) {
  if (g == nullptr) return false;
  int any = 0;
  for (int i = 0; i < n; ++i) any |= g[i];
  return any != 0;
}

template <typename... KArgs, typename... Args>
inline void launch_step(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                        Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ---------------------------------------------------------------------------
// Packed float32 pairs (sm_100 FADD2 / FMUL2): two independent IEEE
// round-to-nearest float32 operations per instruction, no flush-to-zero — each
// lane of the pair is bitwise the scalar __fadd_rn / __fsub_rn / __fmul_rn, so
// they halve the instruction count of the elementwise x/y work without
// touching parity.
// ---------------------------------------------------------------------------
SS_DEV float2 fsub2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
SS_DEV float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
SS_DEV float2 fmul2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// (sqnorm of pair .x, sqnorm of pair .y) for dx = (dx0, dx1), dy = (dy0, dy1).
// NEVER feed fmul2 into fadd2/fsub2: ptxas contracts mul.rn.f32x2 +
// add.rn.f32x2 into FFMA2 even under -fmad=false (checked on nvcc 12.9), which
// would round once instead of twice.  The sums stay scalar (__fadd_rn is
// never contracted); tests/test_native_abi.py asserts the library holds no FFMA2.
SS_DEV float2 sqnorm2(float2 dx, float2 dy) {
  const float2 x2 = fmul2(dx, dx), y2 = fmul2(dy, dy);
  return make_float2(__fadd_rn(x2.x, y2.x), __fadd_rn(x2.y, y2.y));
}

// numpy clip(x, -u, u) with f32 bounds (env.py:97).
SS_DEV float clip_sym(float x, float u) { return fminf(fmaxf(x, -u), u); }

// collision_force (dynamics.py:36-66) for one env: force on i (j gets -f).
// Returns the active flag; inactive pairs contribute nothing.  The activity
// test `norm <= d_min` is decided on the squared distance against
// d2_act = max{x : fl(sqrt(x)) <= d_min} (host-computed, _numerics.py), which
// is exactly equivalent; the square root is only taken for active pairs.
SS_DEV bool contact_force(float pix, float piy, float pjx, float pjy, float dmin, float d2_act,
                          float sign, float ck, float k, float& fx, float& fy) {
  const float x = fsub(pix, pjx);
  const float y = fsub(piy, pjy);
  const float d2 = fadd(fmul(x, x), fmul(y, y));
  if (!(d2 <= d2_act)) { fx = 0.0f; fy = 0.0f; return false; }
  const float d = fsqrt(d2);
  float dx, dy;
  if (d < 1e-8f) { dx = sign; dy = 0.0f; }            // DEGENERATE_DIST, dynamics.py:23
  else { dx = fdiv(x, d); dy = fdiv(y, d); }
  const float mag = fmul(ck, np_softplus(fdiv(fsub(dmin, d), k)));
  fx = fmul(dx, mag);
  fy = fmul(dy, mag);
  return true;
}

// The active-pair part of contact_force (square root, the two divisions,
// the softplus) as ONE out-of-line copy: kernels that would otherwise inline
// it at many call sites (k_flocking_w) keep their hot loop in the
// instruction cache.  Returns the force on i; same arithmetic as above.
static __device__ __noinline__ float2 contact_active(float x, float y, float d2, float dmin, float sign, float ck,
                                              float k) {
  const float d = fsqrt(d2);
  float dx, dy;
  if (d < 1e-8f) { dx = sign; dy = 0.0f; }            // DEGENERATE_DIST, dynamics.py:23
  else { dx = fdiv(x, d); dy = fdiv(y, d); }
  const float mag = fmul(ck, np_softplus(fdiv(fsub(dmin, d), k)));
  return make_float2(fmul(dx, mag), fmul(dy, mag));
}

// contact_force with the active part out of line.
SS_DEV bool contact_force_ol(float pix, float piy, float pjx, float pjy, float dmin, float d2_act,
                             float sign, float ck, float k, float& fx, float& fy) {
  const float x = fsub(pix, pjx);
  const float y = fsub(piy, pjy);
  const float d2 = fadd(fmul(x, x), fmul(y, y));
  if (!(d2 <= d2_act)) { fx = 0.0f; fy = 0.0f; return false; }
  const float2 f = contact_active(x, y, d2, dmin, sign, ck, k);
  fx = f.x;
  fy = f.y;
  return true;
}

// closest_point_on_box (geometry.py:79-100): numpy promotes the wall
// selection to float64 (np.where over two Python floats), so the world-frame
// point is evaluated in double and rounded once when Vec2 casts to float32.
SS_DEV void closest_point_on_box(float px, float py, float bxp, float byp, float ca, float sa,
                                 double hx_d, double hy_d, float& ox, float& oy) {
  const float hx = (float)hx_d, hy = (float)hy_d;
  const float relx = fsub(px, bxp), rely = fsub(py, byp);
  const float qx = fadd(fmul(relx, ca), fmul(rely, sa));
  const float qy = fadd(fmul(-relx, sa), fmul(rely, ca));
  const float cx = fminf(fmaxf(qx, -hx), hx);
  const float cy = fminf(fmaxf(qy, -hy), hy);
  const bool inside = (fabsf(qx) < hx) && (fabsf(qy) < hy);
  double bx, by;
  if (inside) {
    const float gap_x = fsub(hx, fabsf(qx));
    const float gap_y = fsub(hy, fabsf(qy));
    const double wall_x = (qx >= 0.0f) ? hx_d : -hx_d;
    const double wall_y = (qy >= 0.0f) ? hy_d : -hy_d;
    if (gap_x <= gap_y) { bx = wall_x; by = (double)qy; }
    else { bx = (double)qx; by = wall_y; }
  } else {
    bx = (double)cx; by = (double)cy;
  }
  const double cad = (double)ca, sad = (double)sa;
  ox = (float)dsub_rn(dadd_rn((double)bxp, dmul_rn(bx, cad)), dmul_rn(by, sad));
  oy = (float)dadd_rn(dadd_rn((double)byp, dmul_rn(bx, sad)), dmul_rn(by, cad));
}

// integrate (dynamics.py:69-86) + clamp_norm (batching.py:160-171).
SS_DEV void integrate_lin(float& px, float& py, float& vx, float& vy, float fx, float fy,
                          float keep, float inv_m_dt, float dt, float max_speed) {
  vx = fadd(fmul(vx, keep), fmul(fx, inv_m_dt));
  vy = fadd(fmul(vy, keep), fmul(fy, inv_m_dt));
  if (max_speed > 0.0f) {
    const float n = norm2(vx, vy);
    if (n > max_speed) {
      const float s = fdiv(max_speed, n);
      vx = fmul(vx, s);
      vy = fmul(vy, s);
    }
  }
  px = fadd(px, fmul(vx, dt));
  py = fadd(py, fmul(vy, dt));
}

SS_DEV void integrate_ang(float& rot, float& w, float tq, float keep, float inv_i_dt, float dt) {
  w = fadd(fmul(w, keep), fmul(tq, inv_i_dt));
  rot = fadd(rot, fmul(w, dt));
}

}  // namespace ss
