// ss_spread.cu — fused Env.step of simple_spread (scenarios/simple_spread.py):
// the eager register kernel and the opt-in cp.async.bulk pipeline.
#include "ss_bulk.cuh"
#include "ss_small.cuh"

namespace ss {

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
  // physics sub-step (PhysK.substeps; the decoded actions are held).  MS:
  // sub-steps > 1 (separate instantiation: the single reference step keeps
  // its register budget).
  template <bool MS>
  SS_DEV void physics(const float2 (&u)[NA], const SmallArgs& a) {
    float ux[NA], uy[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const SsEntityDesc& d = tmpl_ent(a, i);
      ux[i] = decode_axis(u[i].x, d, a.raw_forces);
      uy[i] = decode_axis(u[i].y, d, a.raw_forces);
      if (a.ph.has_gravity) { ux[i] = fadd(ux[i], d.grav_x); uy[i] = fadd(uy[i], d.grav_y); }
    }
    const int nsub = MS ? a.ph.substeps : 1;
    for (int sub = 0; sub < nsub; ++sub) {
      float fx[NA], fy[NA];
#pragma unroll
      for (int i = 0; i < NA; ++i) { fx[i] = ux[i]; fy[i] = uy[i]; }
      int p = 0;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
#pragma unroll
        for (int j = i + 1; j < NA; ++j, ++p) {
          const SsPairDesc pr = tmpl_pair(a, p);
          float cx, cy;
          if (contact_force(px[i], py[i], px[j], py[j], pr.d_min, pr.d2_act, pr.sign, a.ph.ck, a.ph.k, cx, cy)) {
            fx[i] = fadd(fx[i], cx); fy[i] = fadd(fy[i], cy);
            fx[j] = fsub(fx[j], cx); fy[j] = fsub(fy[j], cy);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const SsEntityDesc& d = tmpl_ent(a, i);
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
  // (8-byte shared stores: rows of 4 NA + 2 floats are 8-byte aligned, and
  // lane offsets 4 (4 NA + 2) l hit distinct bank pairs per half warp)
  SS_DEV void obs_row(int i, float* row) const {
    float2* r2 = reinterpret_cast<float2*>(row);
    r2[0] = make_float2(px[i], py[i]);
    r2[1] = make_float2(vx[i], vy[i]);
    int c = 2;
#pragma unroll
    for (int m = 0; m < NA; ++m) r2[c++] = make_float2(fsub(mx[m], px[i]), fsub(my[m], py[i]));
#pragma unroll
    for (int o = 0; o < NA; ++o) {
      if (o == i) continue;
      r2[c++] = make_float2(fsub(px[o], px[i]), fsub(py[o], py[i]));
    }
  }
};

template <int NA, bool MS>
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
    v.template physics<MS>(u, a);
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
    float* sbuf = nullptr;
    float* row = nullptr;
    const int64_t e0 = e - (threadIdx.x & 31);
    const int nvalid = (int)min((int64_t)32, B - e0);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      sbuf = obs_stage(smem, i, NA, O);
      row = sbuf + (threadIdx.x & 31) * O;
      if (valid) v.obs_row(i, row);
      if (nvalid > 0) obs_flush(a.obs + i * a.obs_stride + e0 * O, nvalid, NA, O, sbuf);
    }
    obs_bulk_drain();
  }
}

// ---------------------------------------------------------------------------
// simple_spread, fused open-loop rollout (SsRolloutIO): the step kernel's
// arithmetic for n_steps consecutive steps with the env's agents (and its
// static markers) held in registers between them — state is read once and
// written once per launch, each step moves only its actions and outputs.
// ---------------------------------------------------------------------------
template <int NA>
__global__ void __launch_bounds__(kSmallThreads, SS_ROLLOUT_MINB) k_simple_spread_rollout(const RolloutArgs r) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  const SmallArgs& a = r.a;
  constexpr int O = SpreadEnv<NA>::O;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = e < B;
  const int64_t e0 = e - (threadIdx.x & 31);
  const int nvalid = (int)min((int64_t)32, B - e0);
  SpreadEnv<NA> v;
  int64_t steps = 0;
  if (valid) {
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const float4 q = a.s.dyn[i * B + e];
      v.px[i] = q.x; v.py[i] = q.y; v.vx[i] = q.z; v.vy[i] = q.w;
      const float2 m = a.s.stat[i * B + e];
      v.mx[i] = m.x; v.my[i] = m.y;
    }
    steps = a.s.step_count[e];
  }
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
    if (valid) {
      v.template physics<false>(u, a);
      steps += 1;
      float rew[NA];
      v.rewards(a, rew);
#pragma unroll
      for (int i = 0; i < NA; ++i) __stcs(r.rew[s] + i * B + e, rew[i]);
      r.done[s][e] = (uint8_t)(steps >= a.ph.max_steps);
    }
    if (s > 0) {   // the previous step's bulk stores must have read the staging
      obs_bulk_drain();
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      float* sbuf = obs_stage(smem, i, NA, O);
      float* row = sbuf + (threadIdx.x & 31) * O;
      if (valid) v.obs_row(i, row);
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
    for (int i = 0; i < NA; ++i) a.s.dyn[i * B + e] = make_float4(v.px[i], v.py[i], v.vx[i], v.vy[i]);
    a.s.step_count[e] = steps;
  }
  obs_bulk_drain();
}

int launch_spread_rollout(World& w, RolloutArgs& r, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const unsigned grid = (unsigned)((w.d.batch + kSmallThreads - 1) / kSmallThreads);
  const size_t shmem = obs_stage_bytes(NA, w.d.obs_dim);
#define SS_CASE(n) case n: launch_step(k_simple_spread_rollout<n>, dim3(grid), dim3(kSmallThreads), shmem, st, r); break;
  switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
  return cuda_status(cudaGetLastError(), "simple_spread rollout launch");
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
    v.template physics<true>(u, a);
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

int launch_spread(World& w, SmallArgs& a, cudaStream_t st) {
  const int NA = w.d.n_agents;
  const int64_t B = w.d.batch;
  const bool ms = a.ph.substeps > 1;   // sub-stepped physics: the MS kernel instantiations
  const size_t shmem = obs_stage_bytes(w.d.n_agents, w.d.obs_dim);
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
  if (rest <= 0) return SS_OK;
  const unsigned g2 = (unsigned)((rest + kSmallThreads - 1) / kSmallThreads);
#define SS_CASE(n)                                                                            \
  case n:                                                                                     \
    if (ms) launch_step(k_simple_spread<n, true>, dim3(g2), dim3(kSmallThreads), shmem, st, a);  \
    else launch_step(k_simple_spread<n, false>, dim3(g2), dim3(kSmallThreads), shmem, st, a);    \
    break;
  switch (NA) { SS_CASE(1) SS_CASE(2) SS_CASE(3) SS_CASE(4) SS_CASE(5) SS_CASE(6) SS_CASE(7) SS_CASE(8) }
#undef SS_CASE
  return cuda_status(cudaGetLastError(), "simple_spread step launch");
}

}  // namespace ss
