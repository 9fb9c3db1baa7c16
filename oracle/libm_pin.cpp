// libm_pin — pins the device's restatement of glibc expf / log1pf (and the
// numpy softplus built on them) to this host's libm.  TEST INFRASTRUCTURE.
//
// Compiles paper_2207_03530_b200/csrc/ss_math.cuh as plain host C++ (the
// very code the kernels run) and compares it bit-for-bit with libm:
//   libm_pin [stride]          sampled sweep (every `stride`-th float)
//   libm_pin 1                 exhaustive over the domains the step uses:
//                              expf on all floats in [-110, 90], log1pf on
//                              all floats in [0, 1] plus sampled elsewhere
// Exit status 0 iff every compared value is bit-identical.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2207_03530_b200/csrc/ss_math.cuh"

static uint32_t bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float fromb(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

int main(int argc, char** argv) {
  const uint64_t stride = argc > 1 ? strtoull(argv[1], nullptr, 10) : 97;
  long bad_exp = 0, n_exp = 0, bad_log = 0, n_log = 0, bad_sp = 0, n_sp = 0;
  for (uint64_t u = 0; u < 0x100000000ULL; u += stride) {
    const float x = fromb((uint32_t)u);
    if (std::isnan(x) || !(x > -110.0f && x < 90.0f)) continue;
    ++n_exp;
    if (bits(expf(x)) != bits(ssm::gl_expf(x))) {
      if (bad_exp < 5) fprintf(stderr, "expf mismatch x=%a libm=%a ours=%a\n", x, expf(x), ssm::gl_expf(x));
      ++bad_exp;
    }
  }
  for (uint64_t u = 0; u <= 0x3f800000ULL; u += stride) {   // [0, 1]: the softplus domain
    const float x = fromb((uint32_t)u);
    ++n_log;
    if (bits(log1pf(x)) != bits(ssm::gl_log1pf(x))) {
      if (bad_log < 5) fprintf(stderr, "log1pf mismatch x=%a\n", x);
      ++bad_log;
    }
  }
  for (uint64_t u = 0x80000000ULL; u < 0xff800000ULL; u += stride * 7 + 1) {   // elsewhere, sampled
    const float x = fromb((uint32_t)u);
    if (std::isnan(x) || x <= -1.0f) continue;
    ++n_log;
    if (bits(log1pf(x)) != bits(ssm::gl_log1pf(x))) ++bad_log;
  }
  for (uint64_t u = 0x3f800001ULL; u < 0x7f800000ULL; u += stride * 7 + 1) {
    const float x = fromb((uint32_t)u);
    ++n_log;
    if (bits(log1pf(x)) != bits(ssm::gl_log1pf(x))) ++bad_log;
  }
  // softplus(z) = z + log1pf(expf(-z)) for z > 0 (numpy npy_logaddexpf(0, z))
  for (uint64_t u = 0; u < 0x7f800000ULL; u += stride) {
    const float z = fromb((uint32_t)u);
    ++n_sp;
    const float want = (z == 0.0f) ? 0.0f + 0.693147180559945309417232121458176568f
                                   : z + log1pf(expf(-z));
    if (bits(want) != bits(ssm::np_softplus(z))) ++bad_sp;
  }
  printf("expf   %ld / %ld mismatches\nlog1pf %ld / %ld mismatches\nsoftplus %ld / %ld mismatches\n",
         bad_exp, n_exp, bad_log, n_log, bad_sp, n_sp);
  return (bad_exp || bad_log || bad_sp) ? 1 : 0;
}
