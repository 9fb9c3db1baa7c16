// ss_large.cu — fused Env.step for the many-agent built-ins (dispersion,
// discovery): one warp per environment, 8 environments per CTA.  Lane l owns
// agents l, l+32, ... (T per lane); the env's positions/velocities and its
// landmarks are staged in shared memory so every lane reads every partner
// with broadcast loads.
//
// Pair forces (discovery, all agent pairs): each lane accumulates the force
// on ITS agent k over partners j in the reference's pair-list order
// (dynamics.py:163-180): pairs (j, k) with j < k subtract f(j,k), then pairs
// (k, j) with j > k add f(k,j) — every f evaluated with the reference's own
// operand order, so the sum is bit-identical without cross-lane traffic.
// Range decisions (contact, coverage, eating) compare squared distances with
// host-computed exact bounds (_numerics.py); square roots are only taken for
// values the reference actually produces (active contacts, reward terms).
//
// Observations are >90% of these steps' HBM bytes.  Every row of agent k is
// "template minus own position": the template (landmarks, all agents,
// eaten flags) is built once per env in shared memory, and the A rows are
// produced as one flattened run of 16-byte chunks — lane l writes chunks
// l, l+32, ... across all rows — straight from registers with streaming
// stores, so each warp store instruction covers 512 contiguous bytes.
#include "ss_internal.cuh"

namespace ss {

constexpr int kLargeWarps = 8;
#ifndef SS_OBS_UNROLL
#define SS_OBS_UNROLL 4
#endif
constexpr int kObsUnroll = SS_OBS_UNROLL;
#ifndef SS_LARGE_MINB
#define SS_LARGE_MINB 5   // resident CTAs (of 8 warps) per SM the register budget targets
#endif
constexpr int kLargeMaxAgents = 128;
constexpr int kLargeMaxLandmarks = 128;

struct LargeArgs {
  DevState s;
  PhysK ph;
  const SsEntityDesc* ents;
  const float2* act[kLargeMaxAgents];
  int64_t act_stride;   // act[k] == act[0] + k * act_stride for every agent (0: no such stride)
  float* obs;
  int64_t obs_stride;
  float* rew;
  uint8_t* done;
  int mode;
  int raw_forces;
  const int* guard;
  int guard_n;          // guard words to OR (SsStepIO.guard_count, >= 1)
  int NA, NL, O;     // agents, landmarks (points / food), obs width
  int W;             // flag words
  float dmin;        // discovery: f32(r_a + r_b)
  float d2_act;      // discovery: squared-distance bound of dmin
  float thr2;        // discovery cover_dist / dispersion eat_dist, squared bound
  int quorum;
  double lo_x, lo_y, range_x, range_y;   // discovery relocation box
};

SS_DEV float warp_min(float v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

// Per-warp shared memory.  tmpl is the observation template:
//   discovery : float2 slots [2 pad][NL landmarks][NA agents]  (lm, pos alias it)
//   dispersion: floats [4 pad][NL x (fx, fy, eaten)]
struct WarpSmem {
  float2* pos;     // [NA]
  float2* vel;     // [NA]
  float2* lm;      // [NL] landmark positions
  float* tmpl;     // template (16-byte aligned)
  float* tmpl_shift;  // discovery: the contact bitmap (NA x u64) of agents_physics
  float* tmp;      // [2*NL] per-landmark scratch
  uint32_t* bits;  // [4] landmark flag words
};

__host__ __device__ inline int round4(int n) { return (n + 3) & ~3; }

// First region: discovery's float2 template [2 + NL + NA], or dispersion's
// float template [4 + 3 NL] followed by its agent positions [NA] (float2).
__host__ __device__ inline int tmpl_floats(int NA, int NL) {
  const int disc = 2 * round4(2 * (2 + NL + NA));   // template + contact bitmap (2 NA floats fit)
  const int disp = round4(4 + 3 * NL) + 2 * NA;
  return round4(disc > disp ? disc : disp);
}

__host__ __device__ inline int warp_floats(int NA, int NL) {
  return tmpl_floats(NA, NL) + round4(2 * NA) /*vel*/ + round4(2 * NL) /*lm*/ + round4(2 * NL) /*tmp*/ + 4;
}

SS_DEV WarpSmem carve(float* base, int NA, int NL, bool discovery) {
  WarpSmem w;
  const int t = tmpl_floats(NA, NL);
  w.tmpl = base;
  w.tmpl_shift = base + round4(2 * (2 + NL + NA));
  float* p = base + t;
  w.vel = reinterpret_cast<float2*>(p);
  p += round4(2 * NA);
  if (discovery) {
    float2* t2 = reinterpret_cast<float2*>(base);
    w.lm = t2 + 2;
    w.pos = t2 + 2 + NL;
  } else {
    w.lm = reinterpret_cast<float2*>(p);
    w.pos = reinterpret_cast<float2*>(base + round4(4 + 3 * NL));
  }
  p += round4(2 * NL);
  w.tmp = p;
  p += round4(2 * NL);
  w.bits = reinterpret_cast<uint32_t*>(p);
  return w;
}

// Load own agents, decode + integrate (pair forces only when PAIRS).
// Leaves post-step positions in sm.pos (or `posbuf`) and velocities in sm.vel.
template <int T, bool PAIRS>
SS_DEV void agents_physics(const LargeArgs& a, float2* pos, float2* vel, int64_t e, float (&px)[T],
                           float (&py)[T], float (&vx)[T], float (&vy)[T],
                           unsigned long long* masks = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t B = a.s.B;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int k = lane + 32 * t;
    if (k < a.NA) {
      const float4 q = a.s.dyn[k * B + e];
      px[t] = q.x; py[t] = q.y; vx[t] = q.z; vy[t] = q.w;
      pos[k] = make_float2(q.x, q.y);
    }
  }
  __syncwarp();
  if (a.mode & SS_DO_PHYSICS) {
    float ux[T], uy[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int k = lane + 32 * t;
      ux[t] = 0.0f; uy[t] = 0.0f;
      if (k < a.NA) {
        const SsEntityDesc& d = a.ents[k];
        // one (A, B, 2) action tensor (the usual case): pointer arithmetic
        // on act[0]; a per-lane index into the parameter table would
        // serialise the constant cache over 32 addresses
        const float2* ak = a.act_stride ? a.act[0] + k * a.act_stride : a.act[k];
        const float2 u = ak[e];
        ux[t] = a.raw_forces ? u.x : fmul(clip_sym(u.x, d.u_range), d.u_mult);
        uy[t] = a.raw_forces ? u.y : fmul(clip_sym(u.y, d.u_range), d.u_mult);
        if (a.ph.has_gravity) { ux[t] = fadd(ux[t], d.grav_x); uy[t] = fadd(uy[t], d.grav_y); }
      }
    }
    // physics sub-steps (PhysK.substeps, 1 = reference): decoded actions held,
    // contacts re-evaluated on the sub-step positions staged in pos[]
    for (int sub = 0; sub < a.ph.substeps; ++sub) {
    float fx[T], fy[T];
#pragma unroll
    for (int t = 0; t < T; ++t) { fx[t] = ux[t]; fy[t] = uy[t]; }
    if (PAIRS && masks != nullptr && a.NA <= 64) {
      // Contact bitmap.  The squared distance is symmetric (a - b == -(b - a)
      // and (-x)^2 == x^2 bitwise), so each unordered pair is tested once:
      // lane l tests rows l and NA-1-l against their higher partners (NA-1
      // tests on every lane) and records an active pair in both agents'
      // 64-bit partner masks.  Each lane then walks its own agents' masks in
      // increasing partner order — the reference's per-entity summation
      // order, (j, k) subtractions for j < k before (k, j) additions — and
      // evaluates the oriented exact contact only for those partners.
      const int NA = a.NA;
      for (int k = lane; k < NA; k += 32) masks[k] = 0ull;
      __syncwarp();
      if (lane < (NA + 1) / 2) {
        const int r1 = lane, r2 = NA - 1 - lane, n1 = NA - 1 - lane;
        const int nt = (r1 == r2) ? n1 : NA - 1;
        const float2 p1 = pos[r1], p2 = pos[r2];
        // tests q and q + 1 side by side in packed float32 pairs
        int q = 0;
#pragma unroll 2
        for (; q + 1 < nt; q += 2) {
          const bool fa = q < n1, fb = q + 1 < n1;
          const int ka = fa ? r1 : r2, kb = fb ? r1 : r2;
          const int ja = fa ? r1 + 1 + q : r2 + 1 + (q - n1);
          const int jb = fb ? r1 + 2 + q : r2 + 2 + (q - n1);
          const float2 pa = fa ? p1 : p2, pb = fb ? p1 : p2;
          const float2 qa = pos[ja], qb = pos[jb];
          const float2 d2 = sqnorm2(fsub2(make_float2(pa.x, pb.x), make_float2(qa.x, qb.x)),
                                    fsub2(make_float2(pa.y, pb.y), make_float2(qa.y, qb.y)));
          if (d2.x <= a.d2_act) { atomicOr(masks + ka, 1ull << ja); atomicOr(masks + ja, 1ull << ka); }
          if (d2.y <= a.d2_act) { atomicOr(masks + kb, 1ull << jb); atomicOr(masks + jb, 1ull << kb); }
        }
        if (q < nt) {
          const bool first = q < n1;
          const int k = first ? r1 : r2;
          const int j = first ? r1 + 1 + q : r2 + 1 + (q - n1);
          const float2 pk = first ? p1 : p2;
          const float2 pj = pos[j];
          if (sqnorm(fsub(pk.x, pj.x), fsub(pk.y, pj.y)) <= a.d2_act) {
            atomicOr(masks + k, 1ull << j);
            atomicOr(masks + j, 1ull << k);
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int k = lane + 32 * t;
        if (k >= NA) continue;
        unsigned long long m = masks[k];
        while (m) {
          const int j = __ffsll((long long)m) - 1;
          m &= m - 1ull;
          const float2 pj = pos[j];
          const float sign = ((j + k) & 1) ? -1.0f : 1.0f;
          float cx, cy;
          if (j < k) {
            contact_force(pj.x, pj.y, px[t], py[t], a.dmin, a.d2_act, sign, a.ph.ck, a.ph.k, cx, cy);
            fx[t] = fsub(fx[t], cx); fy[t] = fsub(fy[t], cy);
          } else {
            contact_force(px[t], py[t], pj.x, pj.y, a.dmin, a.d2_act, sign, a.ph.ck, a.ph.k, cx, cy);
            fx[t] = fadd(fx[t], cx); fy[t] = fadd(fy[t], cy);
          }
        }
      }
    } else if (PAIRS) {
      // The squared distance is symmetric ((-x)^2 == x^2 bitwise), so the
      // activity test runs once per (j, k) on pk - pj; the oriented, exact
      // contact (the reference's operand order) only in the rare active case.
      for (int j = 0; j < a.NA; ++j) {
        const float2 pj = pos[j];
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int k = lane + 32 * t;
          const float x = fsub(px[t], pj.x), y = fsub(py[t], pj.y);
          if (sqnorm(x, y) <= a.d2_act && j != k && k < a.NA) {
            const float sign = ((j + k) & 1) ? -1.0f : 1.0f;
            float cx, cy;
            if (j < k) {
              contact_force(pj.x, pj.y, px[t], py[t], a.dmin, a.d2_act, sign, a.ph.ck, a.ph.k, cx, cy);
              fx[t] = fsub(fx[t], cx); fy[t] = fsub(fy[t], cy);
            } else {
              contact_force(px[t], py[t], pj.x, pj.y, a.dmin, a.d2_act, sign, a.ph.ck, a.ph.k, cx, cy);
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
        pos[k] = make_float2(px[t], py[t]);
        if (sub + 1 == a.ph.substeps) a.s.dyn[k * B + e] = make_float4(px[t], py[t], vx[t], vy[t]);
      }
    }
    __syncwarp();   // sub-step positions staged before the next sub-step reads them
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int k = lane + 32 * t;
    if (k < a.NA) vel[k] = make_float2(vx[t], vy[t]);
  }
  __syncwarp();
}

// Walk the flattened (row, chunk) space: lane handles idx = lane + 32*u.
struct ChunkWalk {
  int r, c;
  float* rowp;
  SS_DEV ChunkWalk(int start, int nch, float* base, int64_t stride) {
    r = start / nch;
    c = start - r * nch;
    rowp = base + r * stride;
  }
  SS_DEV void advance(int nch, int64_t stride) {
    c += 32;
    if (c >= nch) {
      c -= nch; ++r; rowp += stride;
      while (c >= nch) { c -= nch; ++r; rowp += stride; }   // only when nch < 32
    }
  }
};

// ---------------------------------------------------------------------------
// discovery (scenarios/discovery.py)
// ---------------------------------------------------------------------------
// 16-byte chunk c of discovery observation row r (see k_discovery).  With
// SS_DISC_SHIFT the template also exists shifted by one slot (t1[s] =
// t2[s + 1]), so the chunk's two slots are one 16-byte load from t2 (both
// before the row's own agent) or t1 (both after it); only the chunk that
// straddles the skipped slot takes a second load.
#ifndef SS_DISC_SHIFT
#define SS_DISC_SHIFT 1
#endif
SS_DEV float4 disc_chunk(const float2* t2, const float2* t1, const WarpSmem& sm, int first_agent_slot, int r,
                         int c) {
  const int skip = first_agent_slot + r;
  const int s0 = 2 * c, s1 = s0 + 1;
  float2 q0, q1;
  if (SS_DISC_SHIFT) {
    const float4 q = reinterpret_cast<const float4*>(s0 >= skip ? t1 : t2)[c];
    q0 = make_float2(q.x, q.y);
    q1 = s1 == skip ? t1[s1] : make_float2(q.z, q.w);
  } else {
    q0 = t2[s0 + (s0 >= skip)];
    q1 = t2[s1 + (s1 >= skip)];
  }
  const float2 pk = sm.pos[r];
  if (c == 0) {
    const float2 vk = sm.vel[r];
    return make_float4(pk.x, pk.y, vk.x, vk.y);
  }
  const float2 d0 = fsub2(q0, pk), d1 = fsub2(q1, pk);
  return make_float4(d0.x, d0.y, d1.x, d1.y);
}

template <int T, int VEC>
__global__ void __launch_bounds__(32 * kLargeWarps, SS_LARGE_MINB) k_discovery(const LargeArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * kLargeWarps + wid;
  const uint64_t Bg = (uint64_t)a.s.global_batch;
  if ((a.mode & SS_DO_POST) && blockIdx.x == 0 && threadIdx.x == 0) {
    philox_advance(a.s.rng_in, 2ull * (uint64_t)a.NL * Bg, a.s.rng_out);
  }
  if (e >= B) return;
  const WarpSmem sm = carve(smem + wid * warp_floats(a.NA, a.NL), a.NA, a.NL, true);
  for (int i = lane; i < a.NL; i += 32) sm.lm[i] = a.s.stat[i * B + e];
  float px[T], py[T], vx[T], vy[T];
#ifdef SS_NO_PAIR_BITMAP
  agents_physics<T, true>(a, sm.pos, sm.vel, e, px, py, vx, vy);
#else
  agents_physics<T, true>(a, sm.pos, sm.vel, e, px, py, vx, vy,
                          reinterpret_cast<unsigned long long*>(sm.tmpl_shift));
#endif

  int64_t steps = 0;
  if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) {
    steps = a.s.step_count[e];
    if (a.mode & SS_DO_COUNT) { steps += 1; if (lane == 0) a.s.step_count[e] = steps; }
  }
  // post_step (discovery.py:57-71): coverage, then a relocation draw for
  // every env and every point regardless of coverage.
  if (a.mode & SS_DO_POST) {
    const uint64_t eg = (uint64_t)(a.s.env_offset + e);
    for (int l = lane; l < 2 * a.NL; l += 32) {   // one lane per (point, axis) draw
      const int i = l >> 1, axis = l & 1;
      sm.tmp[l] = uniform_f32(philox_draw(a.s.rng_in, (uint64_t)(2 * i + axis) * Bg + eg),
                              axis ? a.lo_y : a.lo_x, axis ? a.range_y : a.range_x);
    }
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
          if (k < a.NA) in = sqnorm(fsub(px[t], pt.x), fsub(py[t], pt.y)) <= a.thr2;
          c += __popc(__ballot_sync(0xffffffffu, in));
        }
        if (c >= a.quorum) bits |= 1u << b;
      }
      if (lane == 0) { a.s.flags[w * B + e] = bits; sm.bits[w] = bits; }
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
    // quorum-th nearest agent distance (np.partition), float64 accumulator;
    // the order statistic is taken on squared distances, then one sqrt.
    int score = 0;
    for (int w = 0; w < a.W; ++w) score += __popc((a.mode & SS_DO_POST) ? sm.bits[w] : a.s.flags[w * B + e]);
    double crowding = 0.0;
    for (int i = 0; i < a.NL; ++i) {
      const float2 pt = sm.lm[i];
      float v[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int k = lane + 32 * t;
        v[t] = (k < a.NA) ? sqnorm(fsub(px[t], pt.x), fsub(py[t], pt.y)) : __int_as_float(0x7f800000);
      }
      float kth = 0.0f;
      for (int r = 0; r < a.quorum; ++r) {
        float mine = v[0];
#pragma unroll
        for (int t = 1; t < T; ++t) mine = fminf(mine, v[t]);
        kth = warp_min(mine);
        const unsigned has = __ballot_sync(0xffffffffu, mine == kth);
        if (lane == __ffs(has) - 1) {
          bool removed = false;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            if (!removed && v[t] == kth) { v[t] = __int_as_float(0x7f800000); removed = true; }
          }
        }
      }
      crowding = dadd_rn(crowding, (double)fsqrt(kth));
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
    // template slots: tmpl2[2 + i] = point_i, tmpl2[2 + NL + o] = a_o
    // Row k skips agent k's own slot: template slot s for s < 2 + NL + k,
    // slot s + 1 beyond it.
    const float2* t2 = reinterpret_cast<const float2*>(sm.tmpl);
    const int first_agent_slot = 2 + a.NL;
    // the one-slot-shifted template, in the contact bitmap's region (free
    // after the physics)
    float2* t1 = reinterpret_cast<float2*>(sm.tmpl_shift);
    if (SS_DISC_SHIFT) {
      for (int k = lane; k < 1 + a.NL + a.NA; k += 32) t1[k] = t2[k + 1];
      __syncwarp();
    }
    if (VEC == 4) {
      // all rows' 16-byte chunks as one flattened run, lane l taking l,
      // l+32, ...; slot s of row k reads template slot s + (s >= 2+NL+k)
      // (row k skips agent k's own slot); chunk 0 is [x, y, vx, vy]
      const int nch = a.O >> 2;
      const int total = a.NA * nch;
      const int64_t stride4 = a.obs_stride >> 2;
      if (nch >= 32) {
        int r = 0, c = lane;                      // lane < 32 <= nch: row 0
        float4* rowp = reinterpret_cast<float4*>(a.obs + e * a.O);
        int idx = lane;
        // kObsUnroll chunks per lane and round: all shared loads first, then
        // the subtractions and streaming stores (latency overlap)
        for (; idx + 32 * (kObsUnroll - 1) < total; idx += 32 * kObsUnroll) {
          float4 v[kObsUnroll];
          float4* dst[kObsUnroll];
#pragma unroll
          for (int u = 0; u < kObsUnroll; ++u) {
            v[u] = disc_chunk(t2, t1, sm, first_agent_slot, r, c);
            dst[u] = rowp + c;
            c += 32;
            if (c >= nch) { c -= nch; ++r; rowp += stride4; }
          }
#pragma unroll
          for (int u = 0; u < kObsUnroll; ++u) __stcs(dst[u], v[u]);
        }
        for (; idx < total; idx += 32) {
          __stcs(rowp + c, disc_chunk(t2, t1, sm, first_agent_slot, r, c));
          c += 32;
          if (c >= nch) { c -= nch; ++r; rowp += stride4; }
        }
      } else {
        for (int idx = lane; idx < total; idx += 32) {
          const int r = idx / nch, c = idx - r * nch;
          __stcs(reinterpret_cast<float4*>(a.obs + r * a.obs_stride + e * a.O) + c,
                 disc_chunk(t2, t1, sm, first_agent_slot, r, c));
        }
      }
    } else {
      const int slots = a.O >> 1;
      const int total = a.NA * slots;
      ChunkWalk w(lane, slots, a.obs + e * a.O, a.obs_stride);
      for (int idx = lane; idx < total; idx += 32) {
        const float2 pk = sm.pos[w.r];
        const int skip = first_agent_slot + w.r;
        const int s = w.c;
        float2 v;
        if (s == 0) v = pk;
        else if (s == 1) v = sm.vel[w.r];
        else {
          const float2 q = t2[s + (s >= skip)];
          v = make_float2(fsub(q.x, pk.x), fsub(q.y, pk.y));
        }
        __stcs(reinterpret_cast<float2*>(w.rowp) + w.c, v);
        w.advance(slots, a.obs_stride);
      }
    }
  }
}

// 16-byte chunk c of dispersion observation row r: chunk c > 0 covers
// template floats 4c..4c+3; element 4c+u belongs to item field (c - 1 + u) % 3:
// 0 -> x (minus own x), 1 -> y, 2 -> eaten flag (minus +0: bitwise unchanged).
SS_DEV float4 disp_chunk(const WarpSmem& sm, const float2* apos, int r, int c) {
  const float2 pk = apos[r];
  if (c == 0) {
    const float2 vk = sm.vel[r];
    return make_float4(pk.x, pk.y, vk.x, vk.y);
  }
  const int m = (c - 1) % 3;
  const float4 t = reinterpret_cast<const float4*>(sm.tmpl)[c];
  const float s0 = m == 0 ? pk.x : (m == 1 ? pk.y : 0.0f);
  const float s1 = m == 0 ? pk.y : (m == 1 ? 0.0f : pk.x);
  const float s2 = m == 0 ? 0.0f : (m == 1 ? pk.x : pk.y);
  const float2 lo = fsub2(make_float2(t.x, t.y), make_float2(s0, s1));
  const float2 hi = fsub2(make_float2(t.z, t.w), make_float2(s2, s0));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// ---------------------------------------------------------------------------
// dispersion (scenarios/dispersion.py): agents non-collidable (no pairs).
// ---------------------------------------------------------------------------
template <int T, int VEC>
__global__ void __launch_bounds__(32 * kLargeWarps, SS_LARGE_MINB) k_dispersion(const LargeArgs a) {
  extern __shared__ __align__(16) float smem[];
  grid_dep_sync();
  if (guard_tripped(a.guard, a.guard_n)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t B = a.s.B;
  const int64_t e = (int64_t)blockIdx.x * kLargeWarps + wid;
  if (e >= B) return;
  const WarpSmem sm = carve(smem + wid * warp_floats(a.NA, a.NL), a.NA, a.NL, false);
  for (int i = lane; i < a.NL; i += 32) sm.lm[i] = a.s.stat[i * B + e];
  float px[T], py[T], vx[T], vy[T];
  float2* apos = sm.pos;
  agents_physics<T, false>(a, apos, sm.vel, e, px, py, vx, vy);

  int64_t steps = 0;
  if (a.mode & (SS_DO_COUNT | SS_DO_DONE)) {
    steps = a.s.step_count[e];
    if (a.mode & SS_DO_COUNT) { steps += 1; if (lane == 0) a.s.step_count[e] = steps; }
  }
  // nearest-agent squared distance per food item: serves post_step's
  // "reached" (any d <= eat_dist  <=>  min d2 <= bound) and the hunger term
  // (sqrt of the min).
  if (a.mode & (SS_DO_POST | SS_DO_REWARD)) {
    // food items i and i + 32 of a lane side by side in packed float32 pairs
    for (int i = lane; i < a.NL; i += 64) {
      const bool two = i + 32 < a.NL;
      const float2 f0 = sm.lm[i], f1 = two ? sm.lm[i + 32] : f0;
      const float2 fx = make_float2(f0.x, f1.x), fy = make_float2(f0.y, f1.y);
      float b0 = __int_as_float(0x7f800000), b1 = b0;
#pragma unroll 4
      for (int j = 0; j < a.NA; ++j) {
        const float2 p = apos[j];
        const float2 d2 = sqnorm2(fsub2(make_float2(p.x, p.x), fx), fsub2(make_float2(p.y, p.y), fy));
        b0 = fminf(b0, d2.x);
        b1 = fminf(b1, d2.y);
      }
      sm.tmp[i] = b0;
      if (two) sm.tmp[i + 32] = b1;
    }
  }
  if (lane < a.W) sm.bits[lane] = a.s.flags[lane * B + e];
  __syncwarp();
  float fresh = 0.0f;
  if (a.mode & SS_DO_POST) {   // dispersion.py:56-66
    int newly = 0;
    for (int w = 0; w < a.W; ++w) {
      const int i = w * 32 + lane;
      const bool reached = (i < a.NL) && (sm.tmp[i] <= a.thr2);
      const uint32_t r = __ballot_sync(0xffffffffu, reached);
      const uint32_t old = sm.bits[w];
      newly += __popc(r & ~old);
      __syncwarp();
      if (lane == 0) { sm.bits[w] = old | r; a.s.flags[w * B + e] = old | r; }
      __syncwarp();
    }
    fresh = (float)newly;
    if (lane == 0) a.s.aux[e] = fresh;
  } else if (a.mode & SS_DO_REWARD) {
    fresh = a.s.aux[e];
  }
  if (a.mode & SS_DO_REWARD) {   // dispersion.py:68-76, float64 hunger in item order
    // the per-item terms (sqrt, cast) in parallel, then lane 0 adds them in
    // item order (the float64 sum is order-sensitive); the terms overwrite
    // the min-d2 scratch: NL doubles exactly fill its 2 NL floats
    float d2v[kLargeMaxLandmarks / 32];
#pragma unroll
    for (int w = 0; w < kLargeMaxLandmarks / 32; ++w) {
      const int i = lane + 32 * w;
      d2v[w] = i < a.NL ? sm.tmp[i] : 0.0f;
    }
    __syncwarp();
    double* term = reinterpret_cast<double*>(sm.tmp);
#pragma unroll
    for (int w = 0; w < kLargeMaxLandmarks / 32; ++w) {
      const int i = lane + 32 * w;
      if (i < a.NL) term[i] = ((sm.bits[w] >> lane) & 1u) ? 0.0 : (double)fsqrt(d2v[w]);
    }
    __syncwarp();
    float r = 0.0f;
    if (lane == 0) {
      double hunger = 0.0;
      for (int i = 0; i < a.NL; ++i) hunger = dadd_rn(hunger, term[i]);
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
    for (int w = 0; w < a.W; ++w) {
      const int n = min(32, a.NL - 32 * w);
      const uint32_t full = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
      all &= (sm.bits[w] & full) == full;
    }
    a.done[e] = (uint8_t)(all | (steps >= a.ph.max_steps));
  }
  if (a.mode & SS_DO_OBS) {
    // row(k) = [x, y, vx, vy, (food_i - a_k, eaten_i)_i]; template
    // tmpl[4 + 3i .. 6 + 3i] = (food_i.x, food_i.y, eaten_i)
    for (int i = lane; i < a.NL; i += 32) {
      const float2 f = sm.lm[i];
      sm.tmpl[4 + 3 * i] = f.x;
      sm.tmpl[5 + 3 * i] = f.y;
      sm.tmpl[6 + 3 * i] = ((sm.bits[i >> 5] >> (i & 31)) & 1u) ? 1.0f : 0.0f;
    }
    __syncwarp();
    const int nch = a.O / VEC;
    const int total = a.NA * nch;
    if (VEC == 4 && nch >= 32) {
      // flattened (row, chunk) run as in k_discovery, kObsUnroll chunks per round
      int r = 0, c = lane;
      float4* rowp = reinterpret_cast<float4*>(a.obs + e * a.O);
      const int64_t stride4 = a.obs_stride >> 2;
      int idx = lane;
      for (; idx + 32 * (kObsUnroll - 1) < total; idx += 32 * kObsUnroll) {
        float4 v[kObsUnroll];
        float4* dst[kObsUnroll];
#pragma unroll
        for (int u = 0; u < kObsUnroll; ++u) {
          v[u] = disp_chunk(sm, apos, r, c);
          dst[u] = rowp + c;
          c += 32;
          if (c >= nch) { c -= nch; ++r; rowp += stride4; }
        }
#pragma unroll
        for (int u = 0; u < kObsUnroll; ++u) __stcs(dst[u], v[u]);
      }
      for (; idx < total; idx += 32) {
        __stcs(rowp + c, disp_chunk(sm, apos, r, c));
        c += 32;
        if (c >= nch) { c -= nch; ++r; rowp += stride4; }
      }
      return;
    }
    ChunkWalk w(lane, nch, a.obs + e * a.O, a.obs_stride);
    for (int idx = lane; idx < total; idx += 32) {
      const float2 pk = apos[w.r];
      if (VEC == 4) {
        __stcs(reinterpret_cast<float4*>(w.rowp) + w.c, disp_chunk(sm, apos, w.r, w.c));
      } else {
        const int j = w.c;
        float x;
        if (j < 4) {
          const float2 vk = sm.vel[w.r];
          x = j == 0 ? pk.x : (j == 1 ? pk.y : (j == 2 ? vk.x : vk.y));
        } else {
          const int t = (j - 4) % 3;
          const float tv = sm.tmpl[j];
          x = t == 0 ? fsub(tv, pk.x) : (t == 1 ? fsub(tv, pk.y) : tv);
        }
        __stcs(w.rowp + j, x);
      }
      w.advance(nch, a.obs_stride);
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
  if (a.NA < 1 || a.NA > kLargeMaxAgents || a.NL > kLargeMaxLandmarks || a.W > 4) {
    set_error("fused many-agent kernel supports up to 128 agents and 128 landmarks");
    return SS_ERR_UNSUPPORTED;
  }
  if (io->mode & SS_DO_PHYSICS) {
    for (int i = 0; i < a.NA; ++i) a.act[i] = reinterpret_cast<const float2*>(io->actions[i]);
    a.act_stride = a.NA > 1 ? a.act[1] - a.act[0] : 0;
    for (int i = 1; i < a.NA && a.act_stride != 0; ++i)
      if (a.act[i] != a.act[0] + i * a.act_stride) a.act_stride = 0;
  }
  a.obs = io->obs;
  a.obs_stride = io->obs_agent_stride;
  a.rew = io->rew;
  a.done = io->done;
  a.mode = io->mode;
  a.raw_forces = io->raw_forces;
  a.guard = io->guard;
  a.guard_n = io->guard_count > 0 ? io->guard_count : 1;
  a.dmin = w.d.sc[0];
  a.d2_act = w.d.sc[2];
  a.thr2 = w.d.sc[3];
  a.quorum = w.d.si[0];
  a.lo_x = w.d.sd[0]; a.lo_y = w.d.sd[1]; a.range_x = w.d.sd[2]; a.range_y = w.d.sd[3];
  const int64_t B = w.d.batch;
  const unsigned grid = (unsigned)((B + kLargeWarps - 1) / kLargeWarps);
  const size_t shmem = (size_t)kLargeWarps * warp_floats(a.NA, a.NL) * sizeof(float);
  const int T = a.NA <= 32 ? 1 : (a.NA <= 64 ? 2 : 4);
  const bool v4 = (a.O % 4) == 0 && (a.obs_stride % 4) == 0;
#define SS_LAUNCH(K)                                                                   \
  do {                                                                                 \
    if (shmem > 48 * 1024)                                                             \
      cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem); \
    launch_step(K, dim3(grid), dim3(32 * kLargeWarps), shmem, st, a);                  \
  } while (0)
  if (w.d.scenario == SS_SCN_DISCOVERY) {
    if (v4) {
      if (T == 1) SS_LAUNCH((k_discovery<1, 4>)); else if (T == 2) SS_LAUNCH((k_discovery<2, 4>)); else SS_LAUNCH((k_discovery<4, 4>));
    } else {
      if (T == 1) SS_LAUNCH((k_discovery<1, 2>)); else if (T == 2) SS_LAUNCH((k_discovery<2, 2>)); else SS_LAUNCH((k_discovery<4, 2>));
    }
  } else {
    if (v4) {
      if (T == 1) SS_LAUNCH((k_dispersion<1, 4>)); else if (T == 2) SS_LAUNCH((k_dispersion<2, 4>)); else SS_LAUNCH((k_dispersion<4, 4>));
    } else {
      if (T == 1) SS_LAUNCH((k_dispersion<1, 1>)); else if (T == 2) SS_LAUNCH((k_dispersion<2, 1>)); else SS_LAUNCH((k_dispersion<4, 1>));
    }
  }
#undef SS_LAUNCH
  return cuda_status(cudaGetLastError(), "fused many-agent step launch");
}

}  // namespace ss
