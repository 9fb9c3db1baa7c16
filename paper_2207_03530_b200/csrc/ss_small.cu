// ss_small.cu — launch_small: fills the SmallArgs of a thread-per-env fused
// step from the world descriptor and dispatches to the kernel family's
// launcher (ss_spread.cu, ss_transport.cu, ss_catalog.cu, ss_flocking.cu).
#include "ss_small.cuh"

namespace ss {

static void fill_const_desc(const World& w, SmallArgs& a) {
  memcpy(a.ek, w.ents.data(), sizeof(SsEntityDesc) * std::min<size_t>(w.ents.size(), kSmallConstEnts));
  memcpy(a.pk, w.pairs.data(), sizeof(SsPairDesc) * std::min<size_t>(w.pairs.size(), kSmallConstPairs));
}

static void fill_small_args(World& w, const SsBuffers* buf, SmallArgs& a) {
  fill_const_desc(w, a);
  a.s = make_state(w, buf);
  a.ph = make_phys(w);
  a.ents = w.d_ents;
  a.pairs = w.d_pairs;
  a.obs_dim = w.d.obs_dim;
  memcpy(a.sc, w.d.sc, sizeof(a.sc));
  memcpy(a.sd, w.d.sd, sizeof(a.sd));
  memcpy(a.si, w.d.si, sizeof(a.si));
  a.E = w.d.n_entities;
  a.P = w.d.n_pairs;
  a.guard_n = 1;
}

// A fused open-loop rollout (SsRolloutIO) — simple_spread and transport /
// reverse_transport, single physics step per Env.step.
// The NaN scans of a rollout's n_steps action sets in one launch (env.py:85
// per step): blockIdx.y = step, a grid-stride pass over that step's agents'
// floats (16-byte streaming loads when aligned), verdict ORed into guard[s].
__global__ void __launch_bounds__(512) k_check_rollout(const RolloutArgs r, int NA, int64_t n, int vec4,
                                                       int* guard) {
  grid_dep_sync();
  const int s = blockIdx.y;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < NA; ++i) {
    if (vec4) {
      // four independent 16-byte loads in flight per thread per trip
      const float4* p = reinterpret_cast<const float4*>(r.act[s][i]);
      const int64_t n4 = n >> 2;
      int64_t k = t0;
      for (; k + 3 * stride < n4; k += 4 * stride) {
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
    } else {
      const float* p = reinterpret_cast<const float*>(r.act[s][i]);
      for (int64_t k = t0; k < n; k += stride) bad |= isnan(p[k]);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(guard + s, 1);
}

static int launch_check_rollout(World& w, const RolloutArgs& r, int* guard, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const int64_t n = 2 * w.d.batch;
  int vec4 = (n % 4) == 0;
  for (int s = 0; s < r.n_steps; ++s)
    for (int i = 0; i < NA; ++i) vec4 &= (reinterpret_cast<uintptr_t>(r.act[s][i]) & 15u) == 0;
  cudaError_t err = cudaMemsetAsync(guard, 0, sizeof(int) * r.n_steps, st);
  if (err != cudaSuccess) return cuda_status(err, "rollout guard reset");
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // ~4 CTAs per SM over all the steps together
  const int64_t per_block = 512LL * (vec4 ? 4 : 1);
  const int64_t want = (n + per_block - 1) / per_block;
  const int64_t cap = (4LL * sms + r.n_steps - 1) / r.n_steps;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min(want, cap));
  launch_step(k_check_rollout, dim3(gx, r.n_steps), dim3(512), 0, st, r, NA, n, vec4, guard);
  return cuda_status(cudaGetLastError(), "rollout action check launch");
}

int launch_rollout(World& w, const SsBuffers* buf, const SsRolloutIO* io, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const bool capable = (w.d.scenario == SS_SCN_SIMPLE_SPREAD || w.d.scenario == SS_SCN_TRANSPORT ||
                        w.d.scenario == SS_SCN_FLOCKING) &&
                       NA >= 1 && NA <= kSmallMaxAgents && w.d.substeps <= 1 && w.d.n_joints == 0;
  if (!capable) {
    set_error("no fused rollout kernel for this world (take the per-step path)");
    return SS_ERR_UNSUPPORTED;
  }
  RolloutArgs r;
  memset(&r, 0, sizeof(r));
  fill_small_args(w, buf, r.a);
  r.a.mode = SS_MODE_STEP;
  r.a.obs_stride = io->obs_agent_stride;
  r.n_steps = io->n_steps;
  for (int s = 0; s < io->n_steps; ++s) {
    for (int i = 0; i < NA; ++i) r.act[s][i] = reinterpret_cast<const float2*>(io->actions[s * NA + i]);
    r.obs[s] = io->obs[s];
    r.rew[s] = io->rew[s];
    r.done[s] = io->done[s];
  }
  r.guard = io->guard;
  if (io->check_actions) {
    const int rc = launch_check_rollout(w, r, io->guard, st);
    if (rc != SS_OK) return rc;
  }
  switch (w.d.scenario) {
    case SS_SCN_SIMPLE_SPREAD: return launch_spread_rollout(w, r, st);
    case SS_SCN_TRANSPORT: return launch_transport_rollout(w, r, st);
    default: return launch_flocking_rollout(w, r, st);
  }
}

int launch_small(World& w, const SsBuffers* buf, const SsStepIO* io, cudaStream_t st) {
  SmallArgs a;
  memset(&a, 0, sizeof(a));
  a.s = make_state(w, buf);
  a.ph = make_phys(w);
  a.ents = w.d_ents;
  a.pairs = w.d_pairs;
  fill_const_desc(w, a);
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
  a.E = w.d.n_entities;
  a.P = w.d.n_pairs;
  switch (w.d.scenario) {
    case SS_SCN_SIMPLE_SPREAD: return launch_spread(w, a, st);
    case SS_SCN_TRANSPORT: return launch_transport(w, a, st);
    case SS_SCN_DROPOUT: return launch_dropout(w, a, st);
    case SS_SCN_WHEEL:
    case SS_SCN_GIVE_WAY:
    case SS_SCN_PASSAGE:
    case SS_SCN_BALANCE:
    case SS_SCN_WATERFALL:
    case SS_SCN_FOOTBALL: return launch_catalog(w, a, st);
    case SS_SCN_FLOCKING: return launch_flocking(w, a, st);
    default:
      set_error("launch_small: not a small scenario");
      return SS_ERR_SCENARIO;
  }
}

}  // namespace ss
