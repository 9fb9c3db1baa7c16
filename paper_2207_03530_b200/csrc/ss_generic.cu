// ss_generic.cu — world_step for arbitrary worlds (dynamics.py:123-184) plus
// the function-level seams (collision_force, closest_points) and the action
// NaN scan.  Used by user-defined scenarios (reward/obs in Python hooks), by
// the catalog scenarios without a fused kernel, and by the module-level
// world_step() API.  One thread per env; the per-entity force/torque
// accumulators of a warp's 32 envs live in shared memory ([E][32] each) so
// any entity count and any pair list run through the same code.
#include "ss_physics.cuh"

namespace ss {

constexpr int kGenericMaxAgents = 256;

struct GenericArgs {
  DevState s;
  PhysK ph;
  const SsEntityDesc* ents;
  const SsPairDesc* pairs;
  const SsJointDesc* joints;
  int E, A, P, J;
  const float2* act[kGenericMaxAgents];
  uint64_t decode_mask[kGenericMaxAgents / 64];  // bit i: decode_action applies
  int mode;
  const int* guard;
  int guard_n;          // guard words to OR (SsStepIO.guard_count, >= 1)
  int* status;   // set to 1 when an unsupported shape pair is met
};

// One thread per env, kGenericThreads per CTA; the per-entity accumulators
// (3 E floats per thread) are the shared-memory footprint.  Two-warp CTAs
// lift the one-warp version's cap of 32 resident CTAs (= 50 % of the SM's
// warps) while small worlds still fit many CTAs per SM.
constexpr int kGenericThreads = 64;

__global__ void __launch_bounds__(kGenericThreads) k_generic_physics(const GenericArgs a) {
  extern __shared__ float sm[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  const int lane = threadIdx.x;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * kGenericThreads + lane;
  if (e >= B) return;
  if (!(a.mode & SS_DO_PHYSICS)) {
    if (a.mode & SS_DO_COUNT) a.s.step_count[e] += 1;
    return;
  }
  // action forces (dynamics.py:151-152); decode_action (env.py:97) when flagged
  const bool ok = env_physics(a.s, a.ph, a.ents, a.pairs, a.E, a.P, a.joints, a.J, a.A, e, sm, kGenericThreads, lane,
                              [&](int i, float& fx, float& fy) {
    if (a.act[i] == nullptr) return false;
    const float2 u = a.act[i][e];
    fx = u.x; fy = u.y;
    if ((a.decode_mask[i >> 6] >> (i & 63)) & 1ull) {
      const SsEntityDesc& d = a.ents[i];
      fx = fmul(clip_sym(u.x, d.u_range), d.u_mult);
      fy = fmul(clip_sym(u.y, d.u_range), d.u_mult);
    }
    return true;
  });
  if (!ok) { *a.status = 1; return; }
  if (a.mode & SS_DO_COUNT) a.s.step_count[e] += 1;
}

int launch_generic(World& w, const SsBuffers* buf, const SsStepIO* io, const uint64_t* decode_mask,
                   int* d_status, cudaStream_t st) {
  GenericArgs a;
  memset(&a, 0, sizeof(a));
  a.s = make_state(w, buf);
  a.ph = make_phys(w);
  a.ents = w.d_ents;
  a.pairs = w.d_pairs;
  a.E = w.d.n_entities;
  a.A = w.d.n_agents;
  a.P = w.d.n_pairs;
  a.joints = w.d_joints;
  a.J = w.d.n_joints;
  if (a.A > kGenericMaxAgents) { set_error("too many agents for world_step"); return SS_ERR_UNSUPPORTED; }
  if (io->mode & SS_DO_PHYSICS) {
    for (int i = 0; i < a.A; ++i) a.act[i] = reinterpret_cast<const float2*>(io->actions[i]);
    for (int i = 0; i < kGenericMaxAgents / 64; ++i) a.decode_mask[i] = decode_mask ? decode_mask[i] : ~0ull;
  }
  a.mode = io->mode;
  a.guard = io->guard;
  a.guard_n = io->guard_count > 0 ? io->guard_count : 1;
  a.status = d_status;
  if (!(io->mode & (SS_DO_PHYSICS | SS_DO_COUNT))) return SS_OK;
  const size_t shmem = (size_t)3 * a.E * kGenericThreads * sizeof(float);
  if (shmem > 200 * 1024) { set_error("world too large for the generic step kernel"); return SS_ERR_UNSUPPORTED; }
  if (shmem > 48 * 1024) {
    cudaFuncSetAttribute(k_generic_physics, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem);
  }
  const unsigned grid = (unsigned)((w.d.batch + kGenericThreads - 1) / kGenericThreads);
  launch_step(k_generic_physics, dim3(grid), dim3(kGenericThreads), shmem, st, a);
  return cuda_status(cudaGetLastError(), "generic world_step launch");
}

// ---- function-level kernels -------------------------------------------------
// largest float x >= 0 with fl(sqrt(x)) <= t (host; mirrors _numerics.py)
float sqrt_le_bound(float t) {
  if (!(t >= 0.0f)) return -1.0f;
  if (isinf(t)) return t;
  float x = t * t;
  while (sqrtf(x) > t) x = nextafterf(x, 0.0f);
  for (;;) {
    const float nx = nextafterf(x, INFINITY);
    if (sqrtf(nx) <= t) x = nx; else return x;
  }
}

__global__ void k_collision_force(const float* pix, const float* piy, const float* pjx,
                                  const float* pjy, float dmin, float d2_act, float sign, float ck,
                                  float k, float* fx, float* fy, uint8_t* active, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x, y;
  active[i] = contact_force(pix[i], piy[i], pjx[i], pjy[i], dmin, d2_act, sign, ck, k, x, y) ? 1 : 0;
  fx[i] = x;
  fy[i] = y;
}

__global__ void k_closest_points(const float2* pos_i, const float* rot_i, ShapeK si,
                                 const float2* pos_j, const float* rot_j, ShapeK sj,
                                 float2* out_i, float2* out_j, int64_t n, int* status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  V2 oi, oj;
  const float2 a = pos_i[i], b = pos_j[i];
  if (!closest_points(v2(a.x, a.y), rot_i[i], si, v2(b.x, b.y), rot_j[i], sj, oi, oj)) {
    *status = 1;
    return;
  }
  out_i[i] = make_float2(oi.x, oi.y);
  out_j[i] = make_float2(oj.x, oj.y);
}

// np.cos / np.sin of a float32 array, bit-exact (ss_math.cuh np_sincosf).
__global__ void k_np_trig(const float* x, float* out, int64_t n, int want_cos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = np_sincosf(x[i], want_cos != 0);
}

int launch_np_trig(const float* x, float* out, int64_t n, int want_cos, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  k_np_trig<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, out, n, want_cos);
  return cuda_status(cudaGetLastError(), "np_trig launch");
}

struct CheckArgs {
  const float* act[kGenericMaxAgents];
  int A;
  int64_t n;   // floats per agent
  int vec4;    // every agent block 16-byte aligned and n % 4 == 0
  int* flag;
};

// NaN scan of every agent's action block (env.py:85): blockIdx.y = agent,
// a grid-stride pass over that agent's floats along x (16-byte loads when
// aligned, four in flight per thread), the verdict ORed into *flag.  About
// 4 CTAs per SM over all the agents together: with A = 64 agents a 1-D grid
// over the agents in turn left each thread ~1 load per agent, 64 dependent
// rounds of memory latency.
__global__ void __launch_bounds__(512) k_check_actions(const CheckArgs a) {
  grid_dep_sync();
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (a.vec4) {
    const int64_t n4 = a.n >> 2;
    const float4* p = reinterpret_cast<const float4*>(a.act[i]);
    if (p != nullptr) {                     // nullptr: a script drives this agent (no raw action)
      int64_t k = t0;
      for (; k + 3 * stride < n4; k += 4 * stride) {   // four 16-byte loads in flight
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldcs(p + k + j * stride);
#pragma unroll
        for (int j = 0; j < 4; ++j) bad |= isnan(v[j].x) | isnan(v[j].y) | isnan(v[j].z) | isnan(v[j].w);
      }
      for (; k < n4; k += stride) {
        const float4 v = __ldcs(p + k);
        bad |= isnan(v.x) | isnan(v.y) | isnan(v.z) | isnan(v.w);
      }
    }
  } else {
    const float* p = a.act[i];
    if (p != nullptr)
      for (int64_t k = t0; k < a.n; k += stride) bad |= isnan(p[k]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flag, 1);
}

int launch_check_actions(int n_agents, int64_t B, const float* const* actions, int* flag,
                         cudaStream_t st) {
  if (n_agents > kGenericMaxAgents) { set_error("too many agents"); return SS_ERR_UNSUPPORTED; }
  if (n_agents == 0) return SS_OK;
  CheckArgs a;
  memset(&a, 0, sizeof(a));
  a.vec4 = ((2 * B) % 4) == 0;
  for (int i = 0; i < n_agents; ++i) {
    a.act[i] = actions[i];
    a.vec4 &= (reinterpret_cast<uintptr_t>(actions[i]) & 15u) == 0;
  }
  a.A = n_agents;
  a.n = 2 * B;
  a.flag = flag;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t per_block = 512LL * (a.vec4 ? 4 : 1);
  const int64_t want = (a.n + per_block - 1) / per_block;   // CTAs one agent's block could use
  const int64_t cap = (4LL * sms + n_agents - 1) / n_agents;  // ~4 CTAs per SM over all agents
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min(want, cap));
  launch_step(k_check_actions, dim3(gx, n_agents), dim3(512), 0, st, a);
  return cuda_status(cudaGetLastError(), "action check launch");
}

// NaN scans of up to SS_MAX_ROLLOUT action sets (the steps of a replay) in
// one launch: blockIdx.y = set * A + agent, a grid-stride pass over that
// agent's floats along x, the verdict ORed into flags[set].
struct SetArgs {
  const float* base[SS_MAX_ROLLOUT];
  int A;
  int64_t agent_stride;   // floats between agent blocks of a set
  int64_t n;              // floats per agent
  int vec4;
  int* flags;
};

__global__ void __launch_bounds__(512) k_check_sets(const SetArgs a) {
  grid_dep_sync();
  const int set = blockIdx.y / a.A, agent = blockIdx.y - set * a.A;
  const float* p = a.base[set] + agent * a.agent_stride;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a.vec4) {
    const float4* p4 = reinterpret_cast<const float4*>(p);
    const int64_t n4 = a.n >> 2;
    int64_t k = t0;
    for (; k + 3 * stride < n4; k += 4 * stride) {
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = __ldcs(p4 + k + j * stride);
#pragma unroll
      for (int j = 0; j < 4; ++j) bad |= isnan(v[j].x) | isnan(v[j].y) | isnan(v[j].z) | isnan(v[j].w);
    }
    for (; k < n4; k += stride) {
      const float4 v = __ldcs(p4 + k);
      bad |= isnan(v.x) | isnan(v.y) | isnan(v.z) | isnan(v.w);
    }
  } else {
    for (int64_t k = t0; k < a.n; k += stride) bad |= isnan(p[k]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags + set, 1);
}

int launch_check_sets(const float* const* bases, int n_sets, int A, int64_t agent_stride, int64_t n,
                      int* flags, cudaStream_t st) {
  SetArgs a;
  memset(&a, 0, sizeof(a));
  a.vec4 = (n % 4) == 0 && (agent_stride % 4) == 0;
  for (int s = 0; s < n_sets; ++s) {
    a.base[s] = bases[s];
    a.vec4 &= (reinterpret_cast<uintptr_t>(bases[s]) & 15u) == 0;
  }
  a.A = A;
  a.agent_stride = agent_stride;
  a.n = n;
  a.flags = flags;
  cudaError_t err = cudaMemsetAsync(flags, 0, sizeof(int) * n_sets, st);
  if (err != cudaSuccess) return cuda_status(err, "action-set flags reset");
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t per_block = 512LL * (a.vec4 ? 4 : 1);
  const int64_t want = (n + per_block - 1) / per_block;
  const int64_t blocks_y = (int64_t)n_sets * A;
  const int64_t cap = (4LL * sms + blocks_y - 1) / blocks_y;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min(want, cap));
  launch_step(k_check_sets, dim3(gx, (unsigned)blocks_y), dim3(512), 0, st, a);
  return cuda_status(cudaGetLastError(), "action-set check launch");
}

// Copy the verdict words into host-mapped memory with plain stores (PCIe
// posted writes; no copy engine).
__global__ void k_publish_flag(const int* flag, int* host_out, int n) {
  grid_dep_sync();
  for (int i = threadIdx.x; i < n; i += blockDim.x) host_out[i] = flag[i];
}

int launch_publish_flag(const int* flag, int* host_out, int n, cudaStream_t st) {
  launch_step(k_publish_flag, dim3(1), dim3(32), 0, st, flag, host_out, n);
  return cuda_status(cudaGetLastError(), "publish_flag launch");
}

int launch_collision_force(const float* pix, const float* piy, const float* pjx, const float* pjy,
                           float dmin, float sign, float ck, float k, float* fx, float* fy,
                           uint8_t* active, int64_t n, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  k_collision_force<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      pix, piy, pjx, pjy, dmin, sqrt_le_bound(dmin), sign, ck, k, fx, fy, active, n);
  return cuda_status(cudaGetLastError(), "collision_force launch");
}

int launch_closest_points(const float* pos_i, const float* rot_i, ShapeK si, const float* pos_j,
                          const float* rot_j, ShapeK sj, float* out_i, float* out_j, int64_t n,
                          int* status, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  k_closest_points<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const float2*>(pos_i), rot_i, si, reinterpret_cast<const float2*>(pos_j),
      rot_j, sj, reinterpret_cast<float2*>(out_i), reinterpret_cast<float2*>(out_j), n, status);
  return cuda_status(cudaGetLastError(), "closest_points launch");
}

}  // namespace ss
