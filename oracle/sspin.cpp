// libsspin.so — the device numerics (paper_2207_03530_b200/csrc/ss_math.cuh)
// compiled as host C++ and exported for the Python pin tests.  TEST
// INFRASTRUCTURE: lets tests compare the kernels' exact restatements of
// numpy float32 sin/cos, glibc expf/log1pf and numpy's Philox stream with
// numpy itself on large samples.
#include <cstdint>

#include "../paper_2207_03530_b200/csrc/ss_math.cuh"

extern "C" {

void pin_np_sincosf(const float* x, float* out, int64_t n, int want_cos) {
  for (int64_t i = 0; i < n; ++i) out[i] = ssm::np_sincosf(x[i], want_cos != 0);
}

void pin_softplus(const float* z, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = ssm::np_softplus(z[i]);
}

// 64-bit draws number idx[i] counted from the 12-word state image
void pin_philox_draw(const uint64_t* state, const uint64_t* idx, uint64_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = ssm::philox_draw(state, idx[i]);
}

void pin_philox_advance(const uint64_t* state, uint64_t n, uint64_t* out) {
  ssm::philox_advance(state, n, out);
}

void pin_uniform_f32(const uint64_t* u, double lo, double range, float* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = ssm::uniform_f32(u[i], lo, range);
}
}
