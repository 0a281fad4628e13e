// Fused router (prefill / batched tokens).
//
// One pass per token computes, from a single read of the residual row h_t:
//   x_t      = bf16(h_t * rsqrt(mean(h_t^2) + eps) * gamma_l)      (written out
//              for the permutation / expert GEMM)
//   p_t      = softmax(x_t . Wg_l^T)            true gate of layer l
//   p^_t     = softmax(x_t . Wg_{l+1}^T)        next-layer prediction (PAPER.md:234,
//              SURVEY a9) -- the 2E gate rows share the x_t read
//   sel_t    = top-k(p_t), ties -> lower id     (moesim/_kernels.py:63-79, bit-exact)
//   w_t      = p_t[sel] / sum p_t[sel]          (Mixtral renormalisation)
//   hist[seq(t), l, e] += 1 for e in sel_t     (metrics.expert_counts, metrics.py:64-71)
//
// Layout: one warp per token (grid-stride), the 2E gate rows staged once per
// CTA in shared memory (2*8*4096*2 B = 128 KB for Mixtral-8x7B), h read as
// float4 (coalesced 512 B per warp instruction).  The router is ~1% of a
// prefill layer (HBM-bound on h: 16 KB/token), so the design goal is
// "one read of h, no extra launches", not tensor cores.
#include "common.cuh"
#include "decide.cuh"

namespace daop {

constexpr int kRouterWarps = 16;
constexpr int kMaxGateRows = 32;  // 2E <= 32  (E <= 16)

struct RouterArgs {
  const float* h;
  const uint16_t* gamma;
  const uint16_t* wg;       // (E, d)
  const uint16_t* wg_next;  // (E, d) or null
  int64_t T;
  int d, E, k;
  float eps;
  uint16_t* x_out;  // (T, d) bf16 or null
  float* p_true;    // (T, E)
  float* p_pred;    // (T, E) or null
  int32_t* topk_idx;
  float* topk_w;
  int32_t* hist;  // per layer slice base or null
  int64_t tokens_per_seq;
  int64_t hist_seq_stride;
};

// softmax over E <= 32 logits held one per lane (max-subtracted, fp32)
static __device__ __forceinline__ float lane_softmax(float z, int lane, int E) {
  float m = lane < E ? z : -INFINITY;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float e = lane < E ? expf(z - m) : 0.f;
  const float s = warp_sum(e);
  return lane < E ? e / s : 0.f;
}

// GATE_IN_SMEM: gate rows staged in shared memory (they fit for d*2E*2 <= ~200 KB)
template <bool GATE_IN_SMEM>
__global__ void __launch_bounds__(kRouterWarps * 32)
    router_kernel(RouterArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int d = a.d, E = a.E;
  const int rows = a.wg_next ? 2 * E : E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ float zscratch[kRouterWarps * kMaxGateRows];
  const uint16_t* gate = nullptr;
  if constexpr (GATE_IN_SMEM) {
    uint4* g = reinterpret_cast<uint4*>(smem);
    const int n16 = E * d / 8;
    const uint4* s0 = reinterpret_cast<const uint4*>(a.wg);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) g[i] = s0[i];
    if (a.wg_next) {
      const uint4* s1 = reinterpret_cast<const uint4*>(a.wg_next);
      for (int i = threadIdx.x; i < n16; i += blockDim.x) g[n16 + i] = s1[i];
    }
    __syncthreads();
    gate = reinterpret_cast<const uint16_t*>(smem);
  }
  const int nchunk = d / 8;  // 8-element chunks, lane-strided
  for (int64_t t = blockIdx.x * (int64_t)kRouterWarps + warp; t < a.T;
       t += (int64_t)gridDim.x * kRouterWarps) {
    const float* hrow = a.h + t * d;
    // pass 1: sum of squares
    float ss = 0.f;
    for (int c = lane; c < nchunk; c += 32) {
      const float4 u = reinterpret_cast<const float4*>(hrow)[2 * c];
      const float4 v = reinterpret_cast<const float4*>(hrow)[2 * c + 1];
      ss = fmaf(u.x, u.x, ss); ss = fmaf(u.y, u.y, ss); ss = fmaf(u.z, u.z, ss); ss = fmaf(u.w, u.w, ss);
      ss = fmaf(v.x, v.x, ss); ss = fmaf(v.y, v.y, ss); ss = fmaf(v.z, v.z, ss); ss = fmaf(v.w, v.w, ss);
    }
    ss = warp_sum(ss);
    const float r = 1.0f / sqrtf(ss / static_cast<float>(d) + a.eps);
    // pass 2: normalise, store x, dot with the gate rows
    float acc[kMaxGateRows];
#pragma unroll
    for (int q = 0; q < kMaxGateRows; ++q) acc[q] = 0.f;
    for (int c = lane; c < nchunk; c += 32) {
      const float4 u = reinterpret_cast<const float4*>(hrow)[2 * c];
      const float4 v = reinterpret_cast<const float4*>(hrow)[2 * c + 1];
      const uint4 gm = reinterpret_cast<const uint4*>(a.gamma)[c];
      const float hv[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
      const uint32_t gw[4] = {gm.x, gm.y, gm.z, gm.w};
      uint32_t xw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float x0 = __fmul_rn(__fmul_rn(hv[2 * q], r), bf16lo(gw[q]));
        const float x1 = __fmul_rn(__fmul_rn(hv[2 * q + 1], r), bf16hi(gw[q]));
        xw[q] = static_cast<uint32_t>(f32_to_bf16_bits(x0)) |
                (static_cast<uint32_t>(f32_to_bf16_bits(x1)) << 16);
      }
      const uint4 x8 = make_uint4(xw[0], xw[1], xw[2], xw[3]);
      if (a.x_out) reinterpret_cast<uint4*>(a.x_out + t * d)[c] = x8;
#pragma unroll
      for (int q = 0; q < kMaxGateRows; ++q) {
        if (q < rows) {
          const uint16_t* grow;
          if constexpr (GATE_IN_SMEM) {
            grow = gate + static_cast<size_t>(q) * d;
          } else {
            grow = (q < E ? a.wg + static_cast<size_t>(q) * d
                          : a.wg_next + static_cast<size_t>(q - E) * d);
          }
          acc[q] = dot8(x8, reinterpret_cast<const uint4*>(grow)[c], acc[q]);
        }
      }
    }
    // reduce in registers, hand the logits to lane 0 through a per-warp smem
    // scratch (taking acc's address would demote it to local memory)
    float* zs = zscratch + warp * kMaxGateRows;
#pragma unroll
    for (int q = 0; q < kMaxGateRows; ++q) {
      if (q < rows) {
        const float z = warp_sum(acc[q]);
        if (lane == 0) zs[q] = z;
      }
    }
    __syncwarp();
    // softmax + top-k + renormalisation, one expert per lane (E <= 16):
    // top-k by (value desc, index asc) == topk_scan / _kernels.py:63-79
    const float p = lane_softmax(lane < E ? zs[lane] : 0.f, lane, E);
    if (lane < E) a.p_true[t * E + lane] = p;
    if (a.wg_next) {
      const float ph = lane_softmax(lane < E ? zs[E + lane] : 0.f, lane, E);
      if (lane < E) a.p_pred[t * E + lane] = ph;
    }
    bool taken = lane >= E;
    int my_sel = -1;
    float my_p = 0.f, den = 0.f;
    for (int j = 0; j < a.k; ++j) {
      float bv = taken ? -INFINITY : p;
      int bi = taken ? 0x7fffffff : lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      den += bv;  // sum of the picked probabilities in pick order (same on all lanes)
      if (lane == j) {
        my_sel = bi;
        my_p = bv;
      }
      if (lane == bi) taken = true;
    }
    if (lane < a.k) {
      a.topk_idx[t * a.k + lane] = my_sel;
      a.topk_w[t * a.k + lane] = my_p / den;
      if (a.hist) atomicAdd(a.hist + (t / a.tokens_per_seq) * a.hist_seq_stride + my_sel, 1);
    }
    __syncwarp();
  }
}

}  // namespace daop

using namespace daop;

extern "C" int daop_router(const float* h, const uint16_t* gamma, const uint16_t* wg,
                           const uint16_t* wg_next, int64_t T, int32_t d, int32_t E, int32_t k,
                           float eps, uint16_t* x_out, float* p_true, float* p_pred,
                           int32_t* topk_idx, float* topk_w, int32_t* hist,
                           int64_t tokens_per_seq, int64_t hist_seq_stride, daop_stream_t st) {
  if (E < 2 || E > kMaxGateRows / 2 || k < 1 || k > E || d % 8 != 0) {
    set_error("router: unsupported shape (E=%d, k=%d, d=%d); needs E <= 16, d %% 8 == 0", E, k, d);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (wg_next && !p_pred) {
    set_error("router: p_pred is required with a next-layer gate");
    return DAOP_ERR_SHAPE;
  }
  if (T == 0) return DAOP_OK;
  if (hist && tokens_per_seq <= 0) tokens_per_seq = T;
  RouterArgs a{h, gamma, wg, wg_next, T, d, E, k, eps, x_out, p_true, p_pred,
               topk_idx, topk_w, hist, tokens_per_seq, hist_seq_stride};
  const int rows = wg_next ? 2 * E : E;
  const size_t smem = static_cast<size_t>(rows) * d * 2;
  int64_t blocks = (T + kRouterWarps - 1) / kRouterWarps;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 2;
  if (smem <= 100 * 1024) {
    if (blocks > cap) blocks = cap;
    DAOP_CUDA(cudaFuncSetAttribute(router_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    router_kernel<true><<<static_cast<int>(blocks), kRouterWarps * 32, smem, as_stream(st)>>>(a);
  } else if (smem <= 200 * 1024 && T >= 4096) {
    const int64_t cap1 = sm_count();
    if (blocks > cap1) blocks = cap1;
    DAOP_CUDA(cudaFuncSetAttribute(router_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    router_kernel<true><<<static_cast<int>(blocks), kRouterWarps * 32, smem, as_stream(st)>>>(a);
  } else {
    if (blocks > cap * 4) blocks = cap * 4;
    router_kernel<false><<<static_cast<int>(blocks), kRouterWarps * 32, 0, as_stream(st)>>>(a);
  }
  DAOP_CHECK_LAUNCH("router");
  return DAOP_OK;
}
