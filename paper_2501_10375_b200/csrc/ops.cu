// Device operator table (replaces moesim/_kernels.py) + device decision
// kernel + random-init fills.
//
//   topk_rows          one thread per row, k passes of the strict '>' scan of
//                      _kernels.py:63-79 (E is tiny: 8-16 in the configs, so a
//                      row fits in registers; rows are the parallel axis).
//   activation_counts  warp-aggregated integer atomics into (L, E) int64,
//                      _kernels.py:94-102 (exact: integer adds commute).
//   pair_overlap       one thread per row, _kernels.py:81-92.
//   plan_layer_f32     decide.cuh plan_layer on device, one thread per token.
#include "common.cuh"
#include "decide.cuh"
#include "rng.cuh"

namespace daop {

template <class S>
__global__ void topk_rows_kernel(const S* __restrict__ s, int64_t n, int e, int k,
                                 int64_t* __restrict__ out) {
  int sel[64];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const S* row = s + r * e;
    int64_t* o = out + r * k;
    if (k <= 64) {
      topk_scan(row, e, k, sel);
      for (int j = 0; j < k; ++j) o[j] = sel[j];
    } else {  // generic path without the register list (k > 64)
      for (int j = 0; j < k; ++j) {
        int best = -1;
        for (int c = 0; c < e; ++c) {
          bool taken = false;
          for (int q = 0; q < j; ++q) taken |= (o[q] == c);
          if (taken) continue;
          if (best < 0 || row[c] > row[best]) best = c;
        }
        o[j] = best;
      }
    }
  }
}

__global__ void activation_counts_kernel(const int64_t* __restrict__ topk, int64_t t, int l, int k,
                                         int e, unsigned long long* __restrict__ counts) {
  const int64_t total = t * l * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int layer = static_cast<int>((i / k) % l);
    const int64_t id = topk[i];
    atomicAdd(counts + static_cast<int64_t>(layer) * e + id, 1ull);
  }
}

__global__ void pair_overlap_kernel(const int64_t* __restrict__ a, const int64_t* __restrict__ b,
                                    int64_t n, int ka, int kb, int64_t* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int x = 0; x < ka; ++x) {
      const int64_t v = a[r * ka + x];
      for (int y = 0; y < kb; ++y) {
        if (v == b[r * kb + y]) {
          ++c;
          break;
        }
      }
    }
    out[r] = c;
  }
}

__global__ void plan_layer_kernel(const float* __restrict__ tr, const float* __restrict__ pp,
                                  const uint8_t* __restrict__ fast_row, int64_t n, int layer, int e,
                                  int k, int start, bool daop_engine, bool graceful,
                                  int32_t* __restrict__ sel, uint8_t* __restrict__ is_fast,
                                  int32_t* __restrict__ drop, int32_t* __restrict__ sub,
                                  int32_t* __restrict__ n_deg) {
  int s_sel[64], s_drop[64], s_sub[64];
  uint8_t s_fast[64];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int nd = plan_layer(layer, tr + t * e, pp ? pp + t * e : nullptr, pp != nullptr,
                              fast_row, e, k, start, daop_engine, graceful, s_sel, s_fast, s_drop,
                              s_sub);
    for (int q = 0; q < k; ++q) {
      sel[t * k + q] = s_sel[q];
      is_fast[t * k + q] = s_fast[q];
      drop[t * k + q] = q < nd ? s_drop[q] : -1;
      sub[t * k + q] = q < nd ? s_sub[q] : -1;
    }
    n_deg[t] = nd;
  }
}

__global__ void fill_bf16_kernel(uint16_t* __restrict__ dst, int64_t n, uint64_t key, float scale,
                                 int64_t off) {
  // 8 elements per thread per iteration, one 16-byte store
  const int64_t n8 = n / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t base = i * 8 + 2 * q;
      uint32_t lo = f32_to_bf16_bits(__fmul_rn(uniform_pm1(key, base + off), scale));
      uint32_t hi = f32_to_bf16_bits(__fmul_rn(uniform_pm1(key, base + 1 + off), scale));
      w[q] = lo | (hi << 16);
    }
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  for (int64_t i = n8 * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = f32_to_bf16_bits(__fmul_rn(uniform_pm1(key, i + off), scale));
}

__global__ void fill_f32_kernel(float* __restrict__ dst, int64_t n, uint64_t key, float scale,
                                int64_t off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __fmul_rn(uniform_pm1(key, i + off), scale);
}

__global__ void fill_norm_kernel(uint16_t* __restrict__ dst, int64_t d, uint64_t key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = f32_to_bf16_bits(__fadd_rn(1.0f, __fmul_rn(0.25f, uniform_pm1(key, i))));
}

static int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 16;
  if (g > cap) g = cap;
  return g < 1 ? 1 : static_cast<int>(g);
}

}  // namespace daop

using namespace daop;

extern "C" {

int daop_topk_rows_f64(const double* s, int64_t n, int32_t e, int32_t k, int64_t* out,
                       daop_stream_t st) {
  if (e < 1 || k < 1 || k > e) {
    set_error("topk_rows: invalid (e=%d, k=%d)", e, k);
    return DAOP_ERR_SHAPE;
  }
  if (n == 0) return DAOP_OK;
  topk_rows_kernel<double><<<grid_for(n, 128), 128, 0, as_stream(st)>>>(s, n, e, k, out);
  DAOP_CHECK_LAUNCH("topk_rows_f64");
  return DAOP_OK;
}

int daop_topk_rows_f32(const float* s, int64_t n, int32_t e, int32_t k, int64_t* out,
                       daop_stream_t st) {
  if (e < 1 || k < 1 || k > e) {
    set_error("topk_rows: invalid (e=%d, k=%d)", e, k);
    return DAOP_ERR_SHAPE;
  }
  if (n == 0) return DAOP_OK;
  topk_rows_kernel<float><<<grid_for(n, 128), 128, 0, as_stream(st)>>>(s, n, e, k, out);
  DAOP_CHECK_LAUNCH("topk_rows_f32");
  return DAOP_OK;
}

int daop_activation_counts(const int64_t* topk, int64_t t, int32_t l, int32_t k, int32_t e,
                           int64_t* counts, daop_stream_t st) {
  const int64_t total = t * l * k;
  if (total == 0) return DAOP_OK;
  activation_counts_kernel<<<grid_for(total, 256), 256, 0, as_stream(st)>>>(
      topk, t, l, k, e, reinterpret_cast<unsigned long long*>(counts));
  DAOP_CHECK_LAUNCH("activation_counts");
  return DAOP_OK;
}

int daop_pair_overlap(const int64_t* a, const int64_t* b, int64_t n, int32_t ka, int32_t kb,
                      int64_t* out, daop_stream_t st) {
  if (n == 0) return DAOP_OK;
  pair_overlap_kernel<<<grid_for(n, 128), 128, 0, as_stream(st)>>>(a, b, n, ka, kb, out);
  DAOP_CHECK_LAUNCH("pair_overlap");
  return DAOP_OK;
}

int daop_plan_layer_f32(const float* tr, const float* pp, const uint8_t* fast_row, int64_t n,
                        int32_t layer, int32_t e, int32_t k, int32_t start, int32_t engine,
                        int32_t graceful, int32_t* sel, uint8_t* is_fast, int32_t* drop,
                        int32_t* sub, int32_t* n_deg, daop_stream_t st) {
  if (e > 64 || k > e || k < 1) {
    set_error("plan_layer: device planner supports E <= 64 (got E=%d, k=%d)", e, k);
    return DAOP_ERR_UNSUPPORTED;
  }
  const bool daop_engine = engine == DAOP_ENGINE_DAOP;
  if (daop_engine && layer >= start && pp == nullptr) {
    set_error("layer %d record carries no prediction for layer %d", layer - 1, layer);
    return DAOP_ERR_PREDICTION_MISSING;
  }
  if (n == 0) return DAOP_OK;
  plan_layer_kernel<<<grid_for(n, 128), 128, 0, as_stream(st)>>>(
      tr, pp, fast_row, n, layer, e, k, start, daop_engine, graceful != 0, sel, is_fast, drop, sub,
      n_deg);
  DAOP_CHECK_LAUNCH("plan_layer_f32");
  return DAOP_OK;
}

int daop_fill_uniform_bf16(uint16_t* dst, int64_t n, uint64_t seed, uint64_t tag, float scale,
                           int64_t off, daop_stream_t st) {
  if (n <= 0) return DAOP_OK;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) != 0) {
    set_error("fill_uniform_bf16: destination must be 16-byte aligned");
    return DAOP_ERR_UNSUPPORTED;
  }
  fill_bf16_kernel<<<grid_for(n / 8 + 1, 256), 256, 0, as_stream(st)>>>(
      dst, n, stream_key(seed, tag), scale, off);
  DAOP_CHECK_LAUNCH("fill_uniform_bf16");
  return DAOP_OK;
}

int daop_fill_uniform_f32(float* dst, int64_t n, uint64_t seed, uint64_t tag, float scale,
                          int64_t off, daop_stream_t st) {
  if (n <= 0) return DAOP_OK;
  fill_f32_kernel<<<grid_for(n, 256), 256, 0, as_stream(st)>>>(dst, n, stream_key(seed, tag),
                                                               scale, off);
  DAOP_CHECK_LAUNCH("fill_uniform_f32");
  return DAOP_OK;
}

int daop_fill_norm_bf16(uint16_t* dst, int64_t d, uint64_t seed, int32_t layer, daop_stream_t st) {
  fill_norm_kernel<<<grid_for(d, 256), 256, 0, as_stream(st)>>>(
      dst, d, stream_key(seed, make_tag(kKindNorm, layer, 0, 0)));
  DAOP_CHECK_LAUNCH("fill_norm_bf16");
  return DAOP_OK;
}

}  // extern "C"
