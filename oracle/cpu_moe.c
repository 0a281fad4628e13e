/* Oracle (TEST / BASELINE INFRASTRUCTURE ONLY): the SwiGLU expert of
 * oracle/numerics.py (expert_act / expert_ffn) in plain C
 * for the CPU baseline bench.py times beside the GPU: bf16 weights as
 * stored (half the bytes of the numpy fp32 restatement), fp32 accumulation,
 * OpenMP over output rows on every host core.  Same arithmetic contract as
 * the numpy oracle (act = bf16(silu(x W1^T) * (x W3^T)), y = act W2^T in
 * fp32); summation order differs, so results agree within the hidden-state
 * tolerance, not bit for bit (tests/test_oracle_cpu.py).
 *
 *   gcc -O3 -march=x86-64-v4 -fopenmp -shared -fPIC cpu_moe.c -o liboracle_cpu.so
 * (built by oracle/build.py; nothing from the product package is used)
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <string.h>

static inline float bf16_to_f32(uint16_t v) {
  uint32_t u = (uint32_t)v << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline float round_bf16(float f) { /* round to nearest even, as numpy oracle rng.round_bf16 */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return f;
}

static inline float dot_bf16(const uint16_t* w, const float* x, int n) {
  float acc[16] = {0};
  int k = 0;
  for (; k + 16 <= n; k += 16)
    for (int i = 0; i < 16; ++i) acc[i] += bf16_to_f32(w[k + i]) * x[k + i];
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i];
  for (; k < n; ++k) s += bf16_to_f32(w[k]) * x[k];
  return s;
}

/* n tokens x (n, d) fp32 (bf16-valued) through one expert: y (n, d) fp32.
 * act (n, ffn) fp32 scratch.  W1, W3 (ffn, d), W2 (d, ffn) bf16 row-major. */
void oracle_expert_ffn(const float* x, int n, const uint16_t* w1, const uint16_t* w3,
                       const uint16_t* w2, int d, int ffn, float* act, float* y) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < ffn; ++r) {
    const uint16_t* a = w1 + (int64_t)r * d;
    const uint16_t* b = w3 + (int64_t)r * d;
    for (int t = 0; t < n; ++t) {
      const float g = dot_bf16(a, x + (int64_t)t * d, d);
      const float u = dot_bf16(b, x + (int64_t)t * d, d);
      act[(int64_t)t * ffn + r] = round_bf16(g / (1.0f + expf(-g)) * u);
    }
  }
#pragma omp parallel for schedule(static)
  for (int r = 0; r < d; ++r) {
    const uint16_t* c = w2 + (int64_t)r * ffn;
    for (int t = 0; t < n; ++t) y[(int64_t)t * d + r] = dot_bf16(c, act + (int64_t)t * ffn, ffn);
  }
}

int oracle_threads(void) { return omp_get_max_threads(); }
