// ss_math.cuh — bit-faithful scalar numerics shared by every kernel.
//
// The reference (swarmsim, pure numpy) computes in float32 with:
//   * separately rounded multiply/add (numpy never contracts to FMA) — the
//     library is compiled with -fmad=false and these helpers use _rn
//     intrinsics so the SASS keeps FMUL/FADD;
//   * IEEE sqrt and division (nvcc defaults -prec-sqrt/-prec-div=true);
//   * np.logaddexp(0, z) for the contact penalty (dynamics.py:59), which in
//     numpy's npymath is  z + log1pf(expf(-z))  with glibc 2.39's expf
//     (x86_64 FMA ifunc variant) and fdlibm log1pf.  Both are restated here
//     and verified bit-exact against this image's libm over every float in
//     the domain used (oracle/libm_pin.c, tests/test_libm_pin.py);
//   * numpy Philox4x64-10 for every random draw (batching.py:174-198) with
//     uniform(lo, hi) = lo + (hi - lo) * ((u >> 11) * 2^-53).
//
// Everything is __host__ __device__ so the host-side pin test compiles the
// very same code with gcc.
#pragma once
#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define SS_HD __host__ __device__ __forceinline__
#else
#define SS_HD static inline
#endif

namespace ssm {

SS_HD uint32_t f2u(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u; memcpy(&u, &f, 4); return u;
#endif
}
SS_HD float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f; memcpy(&f, &u, 4); return f;
#endif
}
SS_HD uint64_t d2u(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u; memcpy(&u, &d, 8); return u;
#endif
}
SS_HD double u2d(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d; memcpy(&d, &u, 8); return d;
#endif
}

// ---- separately rounded float32 / float64 arithmetic -----------------------
#if defined(__CUDA_ARCH__)
SS_HD float fmul(float a, float b) { return __fmul_rn(a, b); }
SS_HD float fadd(float a, float b) { return __fadd_rn(a, b); }
SS_HD float fsub(float a, float b) { return __fsub_rn(a, b); }
SS_HD float fdiv(float a, float b) { return __fdiv_rn(a, b); }
SS_HD float fsqrt(float a) { return __fsqrt_rn(a); }
SS_HD double dmul_rn(double a, double b) { return __dmul_rn(a, b); }
SS_HD double dadd_rn(double a, double b) { return __dadd_rn(a, b); }
SS_HD double dsub_rn(double a, double b) { return __dsub_rn(a, b); }
SS_HD double dfma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
SS_HD float fmul(float a, float b) { return a * b; }
SS_HD float fadd(float a, float b) { return a + b; }
SS_HD float fsub(float a, float b) { return a - b; }
SS_HD float fdiv(float a, float b) { return a / b; }
SS_HD float fsqrt(float a) { return sqrtf(a); }
SS_HD double dmul_rn(double a, double b) { return a * b; }
SS_HD double dadd_rn(double a, double b) { return a + b; }
SS_HD double dsub_rn(double a, double b) { return a - b; }
SS_HD double dfma_rn(double a, double b, double c) { return fma(a, b, c); }
#endif

// x*x + y*y with the reference's rounding (the radicand of Vec2.norm).
SS_HD float sqnorm(float x, float y) { return fadd(fmul(x, x), fmul(y, y)); }
// sqrt(x*x + y*y) exactly as Vec2.norm (batching.py:129-130): no hypot, no FMA.
SS_HD float norm2(float x, float y) { return fsqrt(sqnorm(x, y)); }

// ---- glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, FMA ifunc build) ----
// Table: asuint64(2^(i/32)) - (i << 47), generated from exact decimal powers.
#if defined(__CUDA_ARCH__)
__device__ __constant__
#else
static const
#endif
uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

SS_HD float gl_expf(float x) {
  const double kInvLn2N = 0x1.71547652b82fep+0 * 32.0;
  const double kShift = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0;
  const double C1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0;
  const double C2 = 0x1.62e42ff0c52d6p-1 / 32.0;
  const uint32_t ux = f2u(x);
  const uint32_t abstop = (ux >> 20) & 0x7ffu;
  if (abstop >= (0x42b00000u >> 20)) {            // |x| >= 88 or nan
    if (ux == 0xff800000u) return 0.0f;            // -inf
    if (abstop >= (0x7f800000u >> 20)) return x + x;
    if (x > 0x1.62e42ep6f) return u2f(0x7f800000u);   // overflow -> inf
    if (x < -0x1.9fe368p6f) return 0.0f;               // underflow -> 0
  }
  const double xd = (double)x;
  // gcc -mfma contracts both uses of z = InvLn2N*xd (verified exhaustively).
  double kd = dfma_rn(kInvLn2N, xd, kShift);
  const uint64_t ki = d2u(kd);
  kd = dsub_rn(kd, kShift);
  const double r = dfma_rn(kInvLn2N, xd, -kd);
  uint64_t t = kExp2fTab[ki % 32];
  t += ki << (52 - 5);
  const double s = u2d(t);
  const double z = dfma_rn(C0, r, C1);
  const double r2 = dmul_rn(r, r);
  double y = dfma_rn(C2, r, 1.0);
  y = dfma_rn(z, r2, y);
  y = dmul_rn(y, s);
  return (float)y;
}

// ---- glibc 2.39 log1pf (sysdeps/ieee754/flt-32/s_log1pf.c, fdlibm) ---------
SS_HD float gl_log1pf(float x) {
  const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f;
  const float Lp1 = 6.6666668653e-01f, Lp2 = 4.0000000596e-01f, Lp3 = 2.8571429849e-01f,
              Lp4 = 2.2222198546e-01f, Lp5 = 1.8183572590e-01f, Lp6 = 1.5313838422e-01f,
              Lp7 = 1.4798198640e-01f;
  float hfsq, f = 0.0f, c = 0.0f, s, z, R, u;
  int32_t k, hu = 0;
  const int32_t hx = (int32_t)f2u(x);
  const int32_t ax = hx & 0x7fffffff;
  k = 1;
  if (hx < 0x3ed413d7) {
    if (ax >= 0x3f800000) {
      if (x == -1.0f) return u2f(0xff800000u);
      return u2f(0x7fc00000u);
    }
    if (ax < 0x31000000) {
      if (ax < 0x24800000) return x;
      return fsub(x, fmul(fmul(x, x), 0.5f));
    }
    if (hx > 0 || hx <= (int32_t)0xbe95f61f) { k = 0; f = x; hu = 1; }
  } else if (hx >= 0x7f800000) {
    return x + x;
  }
  if (k != 0) {
    if (hx < 0x5a000000) {
      u = fadd(1.0f, x);
      hu = (int32_t)f2u(u);
      k = (hu >> 23) - 127;
      c = (k > 0) ? fsub(1.0f, fsub(u, x)) : fsub(x, fsub(u, 1.0f));
      c = fdiv(c, u);
    } else {
      u = x;
      hu = (int32_t)f2u(u);
      k = (hu >> 23) - 127;
      c = 0.0f;
    }
    hu &= 0x007fffff;
    if (hu < 0x3504f7) {
      u = u2f((uint32_t)(hu | 0x3f800000));
    } else {
      k += 1;
      u = u2f((uint32_t)(hu | 0x3f000000));
      hu = (0x00800000 - hu) >> 2;
    }
    f = fsub(u, 1.0f);
  }
  hfsq = fmul(fmul(0.5f, f), f);
  const float fk = (float)k;
  if (hu == 0) {
    if (f == 0.0f) {
      if (k == 0) return 0.0f;
      c = fadd(c, fmul(fk, ln2_lo));
      return fadd(fmul(fk, ln2_hi), c);
    }
    R = fmul(hfsq, fsub(1.0f, fmul(0.66666666666666666f, f)));
    if (k == 0) return fsub(f, R);
    return fsub(fmul(fk, ln2_hi), fsub(fsub(R, fadd(fmul(fk, ln2_lo), c)), f));
  }
  s = fdiv(f, fadd(2.0f, f));
  z = fmul(s, s);
  float p = fmul(z, Lp7);
  p = fmul(z, fadd(Lp6, p));
  p = fmul(z, fadd(Lp5, p));
  p = fmul(z, fadd(Lp4, p));
  p = fmul(z, fadd(Lp3, p));
  p = fmul(z, fadd(Lp2, p));
  R = fmul(z, fadd(Lp1, p));
  if (k == 0) return fsub(f, fsub(hfsq, fmul(s, fadd(hfsq, R))));
  return fsub(fmul(fk, ln2_hi),
              fsub(fsub(hfsq, fadd(fmul(s, fadd(hfsq, R)), fadd(fmul(fk, ln2_lo), c))), f));
}

// ---- numpy float32 sin / cos (umath loops_trigonometric, SIMD path) --------
// np.cos / np.sin on float32 arrays (geometry.py:24,32,82) use Cody-Waite
// reduction by pi/2 (3-part constant, fused multiply-adds) and minimax
// polynomials on [-pi/4, pi/4]; |x| beyond the Cody-Waite range falls back to
// libm (approximated here by CUDA's sincosf — such angles never occur in the
// built-in tasks).  Restated from the published algorithm and pinned
// bit-exact against this host's numpy: every float32 in [-71476, 71476]
// (2.4e9 inputs, both functions) and tests/test_numerics_pin.py.
#if defined(__CUDA_ARCH__)
SS_HD float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
#else
SS_HD float ffma(float a, float b, float c) { return fmaf(a, b, c); }
#endif

SS_HD float np_sincosf(float x, bool want_cos) {
  if (x != x) return x;
  const float max_cody = want_cos ? 71476.0625f : 117435.992f;
  if (!(fabsf(x) <= max_cody)) {
#if defined(__CUDA_ARCH__)
    float s, c;
    sincosf(x, &s, &c);
    return want_cos ? c : s;
#else
    return want_cos ? cosf(x) : sinf(x);
#endif
  }
  // rint(x * 2/pi) via the fused add of the 1.5*2^23 magic (as numpy does)
  float q = ffma(x, 0x1.45f306p-1f, 0x1.800000p+23f);
  q = fsub(q, 0x1.800000p+23f);
  float r = ffma(q, -0x1.921fb0p+00f, x);
  r = ffma(q, -0x1.5110b4p-22f, r);
  r = ffma(q, -0x1.846988p-48f, r);
  const float r2 = fmul(r, r);
  float c = ffma(0x1.98e616p-16f, r2, -0x1.6c06dcp-10f);
  c = ffma(c, r2, 0x1.55553cp-05f);
  c = ffma(c, r2, -0x1.000000p-01f);
  c = ffma(c, r2, 0x1.000000p+00f);
  float s = ffma(0x1.7d3bbcp-19f, r2, -0x1.a06bbap-13f);
  s = ffma(s, r2, 0x1.11119ap-07f);
  s = ffma(s, r2, -0x1.555556p-03f);
  s = ffma(s, r2, 0.0f);
  s = ffma(s, r, r);
  int32_t iq = (int32_t)q;          // q is integral here
  if (want_cos) iq += 1;
  float v = ((iq & 1) == 0) ? s : c;
  if ((iq & 2) == 2) v = fsub(0.0f, v);
  return v;
}
SS_HD float np_cosf(float x) { return np_sincosf(x, true); }
SS_HD float np_sinf(float x) { return np_sincosf(x, false); }

// numpy npy_logaddexpf(0.0f, z)  (npymath; called by dynamics.py:59).
SS_HD float np_softplus(float z) {
  const float kLogE2f = 0.693147180559945309417232121458176568f;
  if (0.0f == z) return fadd(0.0f, kLogE2f);
  // numpy's two branches (tmp = 0 - z > 0: 0 + log1p(exp(-tmp)); else
  // z + log1p(exp(tmp))) share one exp / log1p of -|z| (0 - z = -z exactly
  // for finite nonzero z): one code path, no divergence between the signs.
  const float l = gl_log1pf(gl_expf(-fabsf(z)));
  return fadd(z < 0.0f ? 0.0f : z, l);   // NaN z: NaN either way
}

// ---- numpy Philox4x64-10 ----------------------------------------------------
struct U256 { uint64_t w[4]; };

SS_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#if defined(__CUDA_ARCH__)
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

SS_HD U256 philox4x64_10(U256 c, uint64_t k0, uint64_t k1) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c.w[0], &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c.w[2], &hi1, &lo1);
    U256 n;
    n.w[0] = hi1 ^ c.w[1] ^ k0;
    n.w[1] = lo1;
    n.w[2] = hi0 ^ c.w[3] ^ k1;
    n.w[3] = lo0;
    c = n;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  return c;
}

SS_HD U256 u256_add(U256 a, uint64_t b) {
  U256 r = a;
  r.w[0] = a.w[0] + b;
  uint64_t carry = r.w[0] < a.w[0];
  for (int i = 1; i < 4; ++i) {
    r.w[i] = a.w[i] + carry;
    carry = carry && (r.w[i] == 0);
  }
  return r;
}

// Device-resident image of numpy's Philox bit_generator.state.
// words: [0..3] counter, [4..5] key, [6..9] buffer, [10] buffer_pos, [11] spare.
#ifndef SS_RNG_WORDS
#define SS_RNG_WORDS 12
#endif

// 64-bit draw number `n` (0-based) counted from state `st`, identical to the
// n-th call of numpy's philox_next64 starting at that state.
SS_HD uint64_t philox_draw(const uint64_t* st, uint64_t n) {
  const uint64_t pos = st[10];
  const uint64_t left = 4 - pos;          // values remaining in the buffer
  if (n < left) return st[6 + pos + n];
  const uint64_t m = n - left;
  U256 c; c.w[0] = st[0]; c.w[1] = st[1]; c.w[2] = st[2]; c.w[3] = st[3];
  c = u256_add(c, 1 + m / 4);
  const U256 o = philox4x64_10(c, st[4], st[5]);
  return o.w[m % 4];
}

// State after consuming `n` draws (numpy semantics, including the buffer).
SS_HD void philox_advance(const uint64_t* st, uint64_t n, uint64_t* out) {
  for (int i = 0; i < SS_RNG_WORDS; ++i) out[i] = st[i];
  const uint64_t pos = st[10];
  const uint64_t left = 4 - pos;
  if (n <= left) { out[10] = pos + n; return; }
  const uint64_t m = n - left;
  const uint64_t blocks = (m + 3) / 4;
  U256 c; c.w[0] = st[0]; c.w[1] = st[1]; c.w[2] = st[2]; c.w[3] = st[3];
  c = u256_add(c, blocks);
  const U256 o = philox4x64_10(c, st[4], st[5]);
  for (int i = 0; i < 4; ++i) { out[i] = c.w[i]; out[6 + i] = o.w[i]; }
  out[10] = m - 4 * (blocks - 1);
}

// numpy random_uniform: off + scale * next_double (float64).
SS_HD double uniform_f64(uint64_t u, double lo, double range) {
  const double d = (double)(u >> 11) * (1.0 / 9007199254740992.0);
  return dadd_rn(lo, dmul_rn(range, d));
}

// ... then .astype(float32).
SS_HD float uniform_f32(uint64_t u, double lo, double range) { return (float)uniform_f64(u, lo, range); }

}  // namespace ssm
