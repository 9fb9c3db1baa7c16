// ss_large.cu — fused Env.step for the many-agent built-ins (dispersion,
// discovery): one warp per environment, 8 environments per CTA.  Lane l owns
// agents l, l+32, ... (T per lane); the env's positions/velocities are staged
// in shared memory so every lane can read every partner (broadcast loads).
//
// Pair forces (discovery, all agent pairs): each lane accumulates the force
// on ITS agent k over partners j in the reference's pair-list order
// (dynamics.py:163-180): pairs (j, k) with j < k subtract f(j,k), then pairs
// (k, j) with j > k add f(k,j) — every f evaluated with the reference's own
// operand order, so the sum is bit-identical without any cross-lane
// communication.  Observation rows (34.8 KB / 50 KB per env, >90% of the
// step's HBM bytes) are built in shared memory and streamed out with
// coalesced 16-byte stores.
#include "ss_internal.cuh"

namespace ss {

constexpr int kLargeWarps = 8;
constexpr int kLargeMaxAgents = 128;
constexpr int kLargeMaxLandmarks = 128;

struct LargeArgs {
  DevState s;
  PhysK ph;
  const SsEntityDesc* ents;
  const float2* act[kLargeMaxAgents];
  float* obs;
  int64_t obs_stride;
  float* rew;
  uint8_t* done;
  int mode;
  int raw_forces;
  const int* guard;
  int NA, NL, O;    // agents, landmarks (points / food), obs width
  int W;             // flag words
  float dmin;        // discovery: f32(r_a + r_b)
  float thr;         // discovery: f32(cover_dist) | dispersion: f32(eat_dist)
  int quorum;
  double lo_x, lo_y, range_x, range_y;   // discovery relocation box
};

SS_DEV float warp_min(float v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

// Stream a staged row (16-byte aligned smem, O floats) to global memory.
SS_DEV void flush_row(float* __restrict__ dst, const float* __restrict__ row, int O) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) != 0) {
    for (int i = lane; i < O; i += 32) __stcs(dst + i, row[i]);
    __syncwarp();
    return;
  }
  const int n4 = O >> 2;
  float4* d4 = reinterpret_cast<float4*>(dst);
  const float4* s4 = reinterpret_cast<const float4*>(row);
  for (int i = lane; i < n4; i += 32) __stcs(d4 + i, s4[i]);
  for (int i = (n4 << 2) + lane; i < O; i += 32) __stcs(dst + i, row[i]);
  __syncwarp();
}

struct WarpSmem {
  float2* pos;     // [NA]
  float2* vel;     // [NA]
  float2* lm;      // [NL] landmark positions
  float* tmp;      // [2*NL] per-landmark scratch
  uint32_t* bits;  // [4] landmark flag words
  float* row;      // [O] (16-byte aligned)
};

SS_DEV WarpSmem carve(float* base, int NA, int NL, int O) {
  // per-warp footprint, rounded to 16 bytes
  WarpSmem w;
  w.pos = reinterpret_cast<float2*>(base);
  w.vel = w.pos + NA;
  w.lm = w.vel + NA;
  w.tmp = reinterpret_cast<float*>(w.lm + NL);
  w.bits = reinterpret_cast<uint32_t*>(w.tmp + 2 * NL);
  const int used = 4 * NA + 2 * NL + 2 * NL + 4;
  w.row = base + ((used + 3) & ~3);
  return w;
}

__host__ __device__ inline int warp_floats(int NA, int NL, int O) {
  const int used = 4 * NA + 2 * NL + 2 * NL + 4;
  return ((used + 3) & ~3) + ((O + 3) & ~3);
}

// Load own agents, decode + integrate (no pair forces unless PAIRS).
template <int T, bool PAIRS>
SS_DEV void agents_physics(const LargeArgs& a, const WarpSmem& sm, int64_t e, float (&px)[T],
                           float (&py)[T], float (&vx)[T], float (&vy)[T]) {
  const int lane = threadIdx.x & 31;
  const int64_t B = a.s.B;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int k = lane + 32 * t;
    if (k < a.NA) {
      const float4 q = a.s.dyn[k * B + e];
      px[t] = q.x; py[t] = q.y; vx[t] = q.z; vy[t] = q.w;
      sm.pos[k] = make_float2(q.x, q.y);
    }
  }
  __syncwarp();
  if (!(a.mode & SS_DO_PHYSICS)) {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int k = lane + 32 * t;
      if (k < a.NA) sm.vel[k] = make_float2(vx[t], vy[t]);
    }
    __syncwarp();
    return;
  }
  float fx[T], fy[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int k = lane + 32 * t;
    fx[t] = 0.0f; fy[t] = 0.0f;
    if (k < a.NA) {
      const SsEntityDesc& d = a.ents[k];
      const float2 u = a.act[k][e];
      fx[t] = a.raw_forces ? u.x : fmul(clip_sym(u.x, d.u_range), d.u_mult);
      fy[t] = a.raw_forces ? u.y : fmul(clip_sym(u.y, d.u_range), d.u_mult);
      if (a.ph.has_gravity) { fx[t] = fadd(fx[t], d.grav_x); fy[t] = fadd(fy[t], d.grav_y); }
    }
  }
  if (PAIRS) {
    for (int j = 0; j < a.NA; ++j) {
      const float2 pj = sm.pos[j];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int k = lane + 32 * t;
        if (k >= a.NA || j == k) continue;
        const float sign = ((j + k) & 1) ? -1.0f : 1.0f;
        float cx, cy;
        if (j < k) {
          if (contact_force(pj.x, pj.y, px[t], py[t], a.dmin, sign, a.ph.ck, a.ph.k, cx, cy)) {
            fx[t] = fsub(fx[t], cx); fy[t] = fsub(fy[t], cy);
          }
        } else {
          if (contact_force(px[t], py[t], pj.x, pj.y, a.dmin, sign, a.ph.ck, a.ph.k, cx, cy)) {
            fx[t] = fadd(fx[t], cx); fy[t] = fadd(fy[t], cy);
          }
        }
      }
    }
  }
  __syncwarp();   // everyone done reading the pre-step positions
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int k = lane + 32 * t;
    if (k < a.NA) {
      const SsEntityDesc& d = a.ents[k];
      integrate_lin(px[t], py[t], vx[t], vy[t], fx[t], fy[t], a.ph.keep, d.inv_m_dt, a.ph.dt,
                    d.max_speed);
      a.s.dyn[k * B + e] = make_float4(px[t], py[t], vx[t], vy[t]);
      sm.pos[k] = make_float2(px[t], py[t]);
      sm.vel[k] = make_float2(vx[t], vy[t]);
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// discovery (scenarios/discovery.py)
// ---------------------------------------------------------------------------
template <int T>
__global__ void __launch_bounds__(32 * kLargeWarps) k_discovery(const LargeArgs a) {
  extern __shared__ __align__(16) float smem[];
  if (a.guard && *a.guard) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * kLargeWarps + wid;
  const uint64_t Bg = (uint64_t)a.s.global_batch;
  if ((a.mode & SS_DO_POST) && blockIdx.x == 0 && threadIdx.x == 0) {
    philox_advance(a.s.rng_in, 2ull * (uint64_t)a.NL * Bg, a.s.rng_out);
  }
  if (e >= B) return;
  const WarpSmem sm = carve(smem + wid * warp_floats(a.NA, a.NL, a.O), a.NA, a.NL, a.O);
  for (int i = lane; i < a.NL; i += 32) sm.lm[i] = a.s.stat[i * B + e];
  float px[T], py[T], vx[T], vy[T];
  agents_physics<T, true>(a, sm, e, px, py, vx, vy);

  int64_t steps = 0;
  if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) {
    steps = a.s.step_count[e];
    if ((a.mode & SS_DO_COUNT)) { steps += 1; if (lane == 0) a.s.step_count[e] = steps; }
  }
  // post_step (discovery.py:57-71): coverage, then a relocation draw for
  // every env and every point regardless of coverage.
  if (a.mode & SS_DO_POST) {
    const uint64_t eg = (uint64_t)(a.s.env_offset + e);
    // relocation draws for all points, one lane per (point, axis)
    for (int l = lane; l < 2 * a.NL; l += 32) {
      const int i = l >> 1, axis = l & 1;
      sm.tmp[l] = uniform_f32(philox_draw(a.s.rng_in, (uint64_t)(2 * i + axis) * Bg + eg),
                              axis ? a.lo_y : a.lo_x, axis ? a.range_y : a.range_x);
    }
    __syncwarp();
    for (int w = 0; w < a.W; ++w) {
      uint32_t bits = 0u;
      for (int b = 0; b < 32; ++b) {
        const int i = w * 32 + b;
        if (i >= a.NL) break;
        const float2 pt = sm.lm[i];
        int c = 0;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int k = lane + 32 * t;
          bool in = false;
          if (k < a.NA) in = norm2(fsub(px[t], pt.x), fsub(py[t], pt.y)) <= a.thr;
          c += __popc(__ballot_sync(0xffffffffu, in));
        }
        if (c >= a.quorum) bits |= 1u << b;
      }
      if (lane == 0) a.s.flags[w * B + e] = bits;
      sm.bits[w] = bits;
    }
    __syncwarp();
    for (int i = lane; i < a.NL; i += 32) {
      if ((sm.bits[i >> 5] >> (i & 31)) & 1u) {
        const float2 f = make_float2(sm.tmp[2 * i], sm.tmp[2 * i + 1]);
        sm.lm[i] = f;
        a.s.stat[i * B + e] = f;
      }
    }
    __syncwarp();
  }
  if (a.mode & SS_DO_REWARD) {
    // score = #covered (float64); crowding = sum over points of the
    // quorum-th nearest agent distance (np.partition), float64 accumulator.
    int score = 0;
    for (int w = 0; w < a.W; ++w) score += __popc((a.mode & SS_DO_POST) ? sm.bits[w] : a.s.flags[w * B + e]);
    double crowding = 0.0;
    for (int i = 0; i < a.NL; ++i) {
      const float2 pt = sm.lm[i];
      float v[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int k = lane + 32 * t;
        v[t] = (k < a.NA) ? norm2(fsub(px[t], pt.x), fsub(py[t], pt.y)) : __int_as_float(0x7f800000);
      }
      float kth = 0.0f;
      for (int r = 0; r < a.quorum; ++r) {
        float mine = v[0];
#pragma unroll
        for (int t = 1; t < T; ++t) mine = fminf(mine, v[t]);
        kth = warp_min(mine);
        const unsigned has = __ballot_sync(0xffffffffu, mine == kth);
        if (lane == __ffs(has) - 1) {
          bool done_rm = false;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            if (!done_rm && v[t] == kth) { v[t] = __int_as_float(0x7f800000); done_rm = true; }
          }
        }
      }
      crowding = dadd_rn(crowding, (double)kth);
    }
    const float r = (float)dsub_rn((double)score, dmul_rn(0.05, crowding));
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int k = lane + 32 * t;
      if (k < a.NA) __stcs(a.rew + k * B + e, r);
    }
  }
  if ((a.mode & SS_DO_DONE) && lane == 0) a.done[e] = (uint8_t)(steps >= a.ph.max_steps);
  if (a.mode & SS_DO_OBS) {
    // row(k) = [x, y, vx, vy, (point_i - a_k)_i, (a_o - a_k)_{o != k}]
    const int slots = a.O >> 1;
    float2* row2 = reinterpret_cast<float2*>(sm.row);
    for (int k = 0; k < a.NA; ++k) {
      const float2 pk = sm.pos[k];
      for (int q = lane; q < slots; q += 32) {
        float2 v;
        if (q == 0) v = pk;
        else if (q == 1) v = sm.vel[k];
        else if (q < 2 + a.NL) { const float2 p = sm.lm[q - 2]; v = make_float2(fsub(p.x, pk.x), fsub(p.y, pk.y)); }
        else {
          int o = q - 2 - a.NL;
          o += (o >= k);
          const float2 p = sm.pos[o];
          v = make_float2(fsub(p.x, pk.x), fsub(p.y, pk.y));
        }
        row2[q] = v;
      }
      flush_row(a.obs + k * a.obs_stride + e * a.O, sm.row, a.O);
    }
  }
}

// ---------------------------------------------------------------------------
// dispersion (scenarios/dispersion.py): agents non-collidable (no pairs).
// ---------------------------------------------------------------------------
template <int T>
__global__ void __launch_bounds__(32 * kLargeWarps) k_dispersion(const LargeArgs a) {
  extern __shared__ __align__(16) float smem[];
  if (a.guard && *a.guard) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * kLargeWarps + wid;
  if (e >= B) return;
  const WarpSmem sm = carve(smem + wid * warp_floats(a.NA, a.NL, a.O), a.NA, a.NL, a.O);
  for (int i = lane; i < a.NL; i += 32) sm.lm[i] = a.s.stat[i * B + e];
  float px[T], py[T], vx[T], vy[T];
  agents_physics<T, false>(a, sm, e, px, py, vx, vy);

  int64_t steps = 0;
  if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) {
    steps = a.s.step_count[e];
    if ((a.mode & SS_DO_COUNT)) { steps += 1; if (lane == 0) a.s.step_count[e] = steps; }
  }
  // nearest-agent distance per food item: serves both post_step's "reached"
  // (any d <= eat_dist  <=>  min d <= eat_dist) and reward's hunger term.
  if (a.mode & (SS_DO_POST | SS_DO_REWARD)) {
    for (int i = lane; i < a.NL; i += 32) {
      const float2 f = sm.lm[i];
      float best = __int_as_float(0x7f800000);
      for (int j = 0; j < a.NA; ++j) {
        const float2 p = sm.pos[j];
        best = fminf(best, norm2(fsub(p.x, f.x), fsub(p.y, f.y)));
      }
      sm.tmp[i] = best;
    }
    __syncwarp();
  }
  uint32_t* eaten = sm.bits;
  if (lane < a.W) eaten[lane] = a.s.flags[lane * B + e];
  __syncwarp();
  float fresh = 0.0f;
  if (a.mode & SS_DO_POST) {   // dispersion.py:56-66
    int newly = 0;
    for (int w = 0; w < a.W; ++w) {
      const int i = w * 32 + lane;
      const bool reached = (i < a.NL) && (sm.tmp[i] <= a.thr);
      const uint32_t r = __ballot_sync(0xffffffffu, reached);
      const uint32_t old = eaten[w];
      newly += __popc(r & ~old);
      __syncwarp();
      if (lane == 0) { eaten[w] = old | r; a.s.flags[w * B + e] = old | r; }
      __syncwarp();
    }
    fresh = (float)newly;
    if (lane == 0) a.s.aux[e] = fresh;
  } else if (a.mode & SS_DO_REWARD) {
    fresh = a.s.aux[e];
  }
  if (a.mode & SS_DO_REWARD) {   // dispersion.py:68-76, float64 hunger
    float r = 0.0f;
    if (lane == 0) {
      double hunger = 0.0;
      for (int i = 0; i < a.NL; ++i) {
        const bool ate = (eaten[i >> 5] >> (i & 31)) & 1u;
        hunger = dadd_rn(hunger, ate ? 0.0 : (double)sm.tmp[i]);
      }
      r = (float)dsub_rn((double)fresh, dmul_rn(0.05, hunger));
    }
    r = __shfl_sync(0xffffffffu, r, 0);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int k = lane + 32 * t;
      if (k < a.NA) __stcs(a.rew + k * B + e, r);
    }
  }
  if ((a.mode & SS_DO_DONE) && lane == 0) {
    bool all = true;
    for (int i = 0; i < a.NL; ++i) all &= (bool)((eaten[i >> 5] >> (i & 31)) & 1u);
    a.done[e] = (uint8_t)(all | (steps >= a.ph.max_steps));
  }
  if (a.mode & SS_DO_OBS) {
    // row(k) = [x, y, vx, vy, (food_i - a_k, eaten_i)_i]
    for (int k = 0; k < a.NA; ++k) {
      const float2 pk = sm.pos[k];
      if (lane == 0) {
        const float2 vk = sm.vel[k];
        sm.row[0] = pk.x; sm.row[1] = pk.y; sm.row[2] = vk.x; sm.row[3] = vk.y;
      }
      for (int i = lane; i < a.NL; i += 32) {
        const float2 f = sm.lm[i];
        sm.row[4 + 3 * i] = fsub(f.x, pk.x);
        sm.row[5 + 3 * i] = fsub(f.y, pk.y);
        sm.row[6 + 3 * i] = ((eaten[i >> 5] >> (i & 31)) & 1u) ? 1.0f : 0.0f;
      }
      flush_row(a.obs + k * a.obs_stride + e * a.O, sm.row, a.O);
    }
  }
}

int launch_large(World& w, const SsBuffers* buf, const SsStepIO* io, cudaStream_t st) {
  LargeArgs a;
  memset(&a, 0, sizeof(a));
  a.s = make_state(w, buf);
  a.ph = make_phys(w);
  a.ents = w.d_ents;
  a.NA = w.d.n_agents;
  a.NL = w.d.n_stat;
  a.O = w.d.obs_dim;
  a.W = w.d.n_flag_words;
  if (a.NA < 1 || a.NA > kLargeMaxAgents || a.NL > kLargeMaxLandmarks) {
    set_error("fused many-agent kernel supports up to 128 agents and 128 landmarks");
    return SS_ERR_UNSUPPORTED;
  }
  if (io->mode & SS_DO_PHYSICS) {
    for (int i = 0; i < a.NA; ++i) a.act[i] = reinterpret_cast<const float2*>(io->actions[i]);
  }
  a.obs = io->obs;
  a.obs_stride = io->obs_agent_stride;
  a.rew = io->rew;
  a.done = io->done;
  a.mode = io->mode;
  a.raw_forces = io->raw_forces;
  a.guard = io->guard;
  a.dmin = w.d.sc[0];
  a.thr = w.d.sc[1];
  a.quorum = w.d.si[0];
  a.lo_x = w.d.sd[0]; a.lo_y = w.d.sd[1]; a.range_x = w.d.sd[2]; a.range_y = w.d.sd[3];
  const int64_t B = w.d.batch;
  const unsigned grid = (unsigned)((B + kLargeWarps - 1) / kLargeWarps);
  const size_t shmem = (size_t)kLargeWarps * warp_floats(a.NA, a.NL, a.O) * sizeof(float);
  const int T = a.NA <= 32 ? 1 : (a.NA <= 64 ? 2 : 4);
#define SS_LAUNCH(K)                                                                   \
  do {                                                                                 \
    if (shmem > 48 * 1024)                                                             \
      cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem); \
    K<<<grid, 32 * kLargeWarps, shmem, st>>>(a);                                       \
  } while (0)
  if (w.d.scenario == SS_SCN_DISCOVERY) {
    if (T == 1) SS_LAUNCH(k_discovery<1>);
    else if (T == 2) SS_LAUNCH(k_discovery<2>);
    else SS_LAUNCH(k_discovery<4>);
  } else {
    if (T == 1) SS_LAUNCH(k_dispersion<1>);
    else if (T == 2) SS_LAUNCH(k_dispersion<2>);
    else SS_LAUNCH(k_dispersion<4>);
  }
#undef SS_LAUNCH
  return cuda_status(cudaGetLastError(), "fused many-agent step launch");
}

}  // namespace ss
