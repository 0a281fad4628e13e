// Non-MoE block of a Mixtral-shaped decoder layer for one decode token
// (the real caller of the MoE block; PAPER.md:110-114:
// "each featuring self-attention, expert layers, normalization, and residual
// connections"; the reference prices it as t_nonmoe, moesim/simulator.py:291).
//
//   xa   = bf16( rmsnorm(h) * gamma_attn )
//   qkv  = xa . Wqkv^T                         fp32, Wqkv = [Wq; Wk; Wv] (q + 2 kv, d)
//   q, k = RoPE(pos) (rotate-half pairs (i, i + hd/2), theta^(-2i/hd), fp32)
//   cache[pos] = bf16(k), bf16(v)              per-layer KV cache (n_kv, max_seq, hd)
//   o_h  = softmax_p(q_h . k_p / sqrt(hd)) . v_p  over p <= pos, GQA (head h uses kv h / group)
//   h'   = h + bf16(o) . Wo^T                  fp32
//
// Four launches, each HBM-bound on what it streams:
//   attn_qkv_kernel      RMSNorm in every CTA + warp-per-row GEMV over Wqkv (50 MB at 8x7B)
//   attn_decode_kernel   flash-decoding: CTA = (kv head, position split), a thread per
//                        position for the scores of the group's q heads (k read once),
//                        a thread per head dim for P.V, online softmax across tiles
//   attn_combine_kernel  per q head, the splits merged in fixed order -> bf16 o
//   attn_oproj_kernel    warp-per-row GEMV over Wo (33.5 MB) + residual
#include "common.cuh"

namespace daop {

constexpr int AT_WARPS = 16;    // GEMV CTAs
constexpr int AT_HD = 128;      // head dim (Mixtral / Llama)
constexpr int AT_TILE = 128;    // positions per attention tile (one per thread)
constexpr int AT_MAX_GROUP = 8; // q heads per kv head

// dot of one bf16 row (K elements, K % 256 == 0) with x (bf16, smem), lane-
// strided 16-byte pieces in fixed order, then a butterfly warp sum
__device__ __forceinline__ float row_dot(const uint16_t* __restrict__ w, const uint4* x_s, int K,
                                         int lane) {
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const int n16 = K / 8;
  float acc = 0.f;
  for (int c0 = 0; c0 < n16; c0 += 32 * 8) {
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = c0 + i * 32 + lane;
      v[i] = c < n16 ? ldg_nc_v4(wr + c) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = c0 + i * 32 + lane;
      if (c < n16) acc = dot8(x_s[c], v[i], acc);
    }
  }
  return warp_sum(acc);
}

// every CTA: xa = bf16(rmsnorm(h) * gamma) into shared memory (fixed-order
// block reduction -> identical in every CTA); CTA 0 also writes it out
__device__ void rmsnorm_to_smem(const float* __restrict__ h, const uint16_t* __restrict__ gamma,
                                int d, float eps, uint16_t* xs, float* red, uint16_t* x_out) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  float ss = 0.f;
  for (int i = tid; i < d; i += nt) ss = fmaf(h[i], h[i], ss);
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    float t = 0.f;
    for (int w = 0; w < nt / 32; ++w) t += red[w];
    red[32] = 1.0f / sqrtf(t / static_cast<float>(d) + eps);
  }
  __syncthreads();
  const float r = red[32];
  for (int i = tid; i < d; i += nt) {
    const uint16_t g = gamma[i];
    const float x = __fmul_rn(__fmul_rn(h[i], r), __uint_as_float(static_cast<uint32_t>(g) << 16));
    xs[i] = f32_to_bf16_bits(x);
    if (x_out && blockIdx.x == 0) x_out[i] = xs[i];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(AT_WARPS * 32, 1)
    attn_qkv_kernel(const float* __restrict__ h, const uint16_t* __restrict__ gamma,
                    const uint16_t* __restrict__ wqkv, int d, int rows, float eps,
                    uint16_t* __restrict__ xa_out, float* __restrict__ qkv) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint16_t* xs = reinterpret_cast<uint16_t*>(smem);
  float* red = reinterpret_cast<float*>(smem + static_cast<size_t>(d) * 2);
  rmsnorm_to_smem(h, gamma, d, eps, xs, red, xa_out);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * AT_WARPS + (threadIdx.x >> 5), nw = gridDim.x * AT_WARPS;
  for (int r = gw; r < rows; r += nw) {
    const float v = row_dot(wqkv + static_cast<int64_t>(r) * d, reinterpret_cast<const uint4*>(xs),
                            d, lane);
    if (lane == 0) qkv[r] = v;
  }
}

// RoPE of one head vector held as hd floats in smem (pairs (i, i + hd/2))
__device__ __forceinline__ void rope_pair(float& a, float& b, int i, int pos, float theta) {
  const float inv = 1.0f / powf(theta, static_cast<float>(2 * i) / static_cast<float>(AT_HD));
  const float ang = static_cast<float>(pos) * inv;
  float s, c;
  sincosf(ang, &s, &c);
  const float a2 = a * c - b * s;
  const float b2 = b * c + a * s;
  a = a2;
  b = b2;
}

struct AttnArgs {
  const float* qkv;       // raw projections: q (n_heads*hd) | k (n_kv*hd) | v (n_kv*hd)
  uint16_t* k_cache;      // (n_kv, max_seq, hd) bf16, this layer
  uint16_t* v_cache;
  int n_heads, n_kv, max_seq, pos, splits, per_split;
  float theta, scale;
  float* part;            // (n_kv, splits, group, 2 + hd): m, l, acc[hd]
};

__global__ void __launch_bounds__(AT_TILE, 1) attn_decode_kernel(AttnArgs a) {
  __shared__ float q_s[AT_MAX_GROUP][AT_HD];
  __shared__ float p_s[AT_MAX_GROUP][AT_TILE];
  __shared__ float red[AT_MAX_GROUP][AT_TILE / 32];
  __shared__ float m_s[AT_MAX_GROUP], l_s[AT_MAX_GROUP], corr_s[AT_MAX_GROUP];
  const int g = blockIdx.x, split = blockIdx.y, tid = threadIdx.x, lane = tid & 31,
            warp = tid >> 5;
  const int group = a.n_heads / a.n_kv;
  const int q_dim = a.n_heads * AT_HD, kv_dim = a.n_kv * AT_HD;
  // q of the group's heads with RoPE (redundant per CTA: 4 x 128 floats)
  for (int i = tid; i < group * (AT_HD / 2); i += blockDim.x) {
    const int hh = i / (AT_HD / 2), j = i - hh * (AT_HD / 2);
    float x0 = a.qkv[(g * group + hh) * AT_HD + j];
    float x1 = a.qkv[(g * group + hh) * AT_HD + j + AT_HD / 2];
    rope_pair(x0, x1, j, a.pos, a.theta);
    q_s[hh][j] = x0;
    q_s[hh][j + AT_HD / 2] = x1;
  }
  const int p0 = split * a.per_split;
  const int p1 = min(a.pos + 1, p0 + a.per_split);
  uint16_t* kc = a.k_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  uint16_t* vc = a.v_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  if (a.pos >= p0 && a.pos < p1) {  // this split holds the new position: append k, v
    for (int j = tid; j < AT_HD / 2; j += blockDim.x) {
      float k0 = a.qkv[q_dim + g * AT_HD + j];
      float k1 = a.qkv[q_dim + g * AT_HD + j + AT_HD / 2];
      rope_pair(k0, k1, j, a.pos, a.theta);
      kc[static_cast<int64_t>(a.pos) * AT_HD + j] = f32_to_bf16_bits(k0);
      kc[static_cast<int64_t>(a.pos) * AT_HD + j + AT_HD / 2] = f32_to_bf16_bits(k1);
    }
    for (int j = tid; j < AT_HD; j += blockDim.x)
      vc[static_cast<int64_t>(a.pos) * AT_HD + j] =
          f32_to_bf16_bits(a.qkv[q_dim + kv_dim + g * AT_HD + j]);
    __threadfence_block();
  }
  if (tid < group) {
    m_s[tid] = -INFINITY;
    l_s[tid] = 0.f;
  }
  __syncthreads();
  float acc[AT_MAX_GROUP];  // thread tid owns head dim tid of every group head
#pragma unroll
  for (int hh = 0; hh < AT_MAX_GROUP; ++hh) acc[hh] = 0.f;
  for (int t0 = p0; t0 < p1; t0 += AT_TILE) {
    const int p = t0 + tid;
    // scores: thread = position, k row read once for the whole group
    float sc[AT_MAX_GROUP];
#pragma unroll
    for (int hh = 0; hh < AT_MAX_GROUP; ++hh) sc[hh] = -INFINITY;
    if (p < p1) {
      const uint4* kr = reinterpret_cast<const uint4*>(kc + static_cast<int64_t>(p) * AT_HD);
      float s[AT_MAX_GROUP];
#pragma unroll
      for (int hh = 0; hh < AT_MAX_GROUP; ++hh) s[hh] = 0.f;
#pragma unroll 4
      for (int c = 0; c < AT_HD / 8; ++c) {
        const uint4 kv = kr[c];
        const uint32_t w4[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float lo = bf16lo(w4[e]), hi = bf16hi(w4[e]);
#pragma unroll
          for (int hh = 0; hh < AT_MAX_GROUP; ++hh)
            if (hh < group) {
              s[hh] = fmaf(q_s[hh][c * 8 + 2 * e], lo, s[hh]);
              s[hh] = fmaf(q_s[hh][c * 8 + 2 * e + 1], hi, s[hh]);
            }
        }
      }
#pragma unroll
      for (int hh = 0; hh < AT_MAX_GROUP; ++hh) sc[hh] = s[hh] * a.scale;
    }
    // tile max per head (fixed-order block reduction)
#pragma unroll
    for (int hh = 0; hh < AT_MAX_GROUP; ++hh) {
      if (hh >= group) break;
      float mx = sc[hh];
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) red[hh][warp] = mx;
    }
    __syncthreads();
    if (tid < group) {
      float mx = -INFINITY;
      for (int w = 0; w < AT_TILE / 32; ++w) mx = fmaxf(mx, red[tid][w]);
      const float mnew = fmaxf(m_s[tid], mx);
      corr_s[tid] = expf(m_s[tid] - mnew);  // 0 on the first tile (m = -inf)
      m_s[tid] = mnew;
    }
    __syncthreads();
#pragma unroll
    for (int hh = 0; hh < AT_MAX_GROUP; ++hh) {
      if (hh >= group) break;
      const float e = p < p1 ? expf(sc[hh] - m_s[hh]) : 0.f;
      p_s[hh][tid] = e;
      const float se = warp_sum(e);
      if (lane == 0) red[hh][warp] = se;
    }
    __syncthreads();
    if (tid < group) {
      float se = 0.f;
      for (int w = 0; w < AT_TILE / 32; ++w) se += red[tid][w];
      l_s[tid] = l_s[tid] * corr_s[tid] + se;
    }
    // P.V: thread = head dim; v rows read coalesced (256 B per position)
#pragma unroll
    for (int hh = 0; hh < AT_MAX_GROUP; ++hh) acc[hh] *= (hh < group ? corr_s[hh] : 1.f);
    const int n = min(AT_TILE, p1 - t0);
#pragma unroll 8
    for (int i = 0; i < n; ++i) {
      const float v = __uint_as_float(static_cast<uint32_t>(
                          vc[static_cast<int64_t>(t0 + i) * AT_HD + tid]) << 16);
#pragma unroll
      for (int hh = 0; hh < AT_MAX_GROUP; ++hh)
        if (hh < group) acc[hh] = fmaf(p_s[hh][i], v, acc[hh]);
    }
    __syncthreads();
  }
  // partial of this split: (m, l, acc)
  for (int hh = 0; hh < group; ++hh) {
    float* pr = a.part + ((static_cast<int64_t>(g) * a.splits + split) * group + hh) * (2 + AT_HD);
    if (tid == 0) {
      pr[0] = m_s[hh];
      pr[1] = l_s[hh];
    }
    pr[2 + tid] = acc[hh];
  }
}

// per q head: merge the splits in fixed order -> o (bf16)
__global__ void attn_combine_kernel(const float* __restrict__ part, int n_heads, int n_kv,
                                    int splits, int used, uint16_t* __restrict__ o) {
  const int head = blockIdx.x, tid = threadIdx.x;
  const int group = n_heads / n_kv, g = head / group, hh = head - g * group;
  float m = -INFINITY;
  for (int s = 0; s < used; ++s)
    m = fmaxf(m, part[((static_cast<int64_t>(g) * splits + s) * group + hh) * (2 + AT_HD)]);
  float l = 0.f, acc = 0.f;
  for (int s = 0; s < used; ++s) {
    const float* pr = part + ((static_cast<int64_t>(g) * splits + s) * group + hh) * (2 + AT_HD);
    const float c = expf(pr[0] - m);
    l = fmaf(pr[1], c, l);
    acc = fmaf(pr[2 + tid], c, acc);
  }
  o[head * AT_HD + tid] = f32_to_bf16_bits(acc / l);
}

// h' = h + o . Wo^T  (rows of Wo are output dims; o bf16 (q_dim) in smem)
__global__ void __launch_bounds__(AT_WARPS * 32, 1)
    attn_oproj_kernel(const float* __restrict__ h, const uint16_t* __restrict__ o,
                      const uint16_t* __restrict__ wo, int d, int q_dim,
                      float* __restrict__ h_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint4* os = reinterpret_cast<uint4*>(smem);
  for (int i = threadIdx.x; i < q_dim / 8; i += blockDim.x)
    os[i] = reinterpret_cast<const uint4*>(o)[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * AT_WARPS + (threadIdx.x >> 5), nw = gridDim.x * AT_WARPS;
  for (int r = gw; r < d; r += nw) {
    const float v = row_dot(wo + static_cast<int64_t>(r) * q_dim, os, q_dim, lane);
    if (lane == 0) h_out[r] = h[r] + v;
  }
}

}  // namespace daop

using namespace daop;

extern "C" int daop_attn_workspace(int32_t n_heads, int32_t n_kv, int32_t max_seq,
                                   int64_t* h_bytes) {
  // qkv fp32 | partials (n_kv x splits(<=64) x group x (2 + hd)) | o bf16
  const int64_t q_dim = static_cast<int64_t>(n_heads) * AT_HD;
  const int64_t kv_dim = static_cast<int64_t>(n_kv) * AT_HD;
  const int64_t part = static_cast<int64_t>(n_kv) * 64 * (n_heads / n_kv) * (2 + AT_HD) * 4;
  *h_bytes = (q_dim + 2 * kv_dim) * 4 + part + q_dim * 2 + 256;
  (void)max_seq;
  return DAOP_OK;
}

extern "C" int daop_attn_decode(const float* d_h, const uint16_t* d_gamma, const uint16_t* d_wqkv,
                                const uint16_t* d_wo, uint16_t* d_k_cache, uint16_t* d_v_cache,
                                int32_t d, int32_t n_heads, int32_t n_kv, int32_t max_seq,
                                int32_t pos, float eps, float theta, uint16_t* d_xa_out,
                                float* d_h_out, void* d_workspace, daop_stream_t stream) {
  const int q_dim = n_heads * AT_HD, kv_dim = n_kv * AT_HD;
  if (n_kv < 1 || n_heads % n_kv != 0 || n_heads / n_kv > AT_MAX_GROUP || d % 256 != 0 ||
      q_dim % 256 != 0 || pos < 0 || pos >= max_seq) {
    set_error("attention: unsupported shape (d=%d heads=%d kv=%d pos=%d max_seq=%d); needs "
              "head_dim 128, d %% 256 == 0, heads/kv <= %d, 0 <= pos < max_seq",
              d, n_heads, n_kv, pos, max_seq, AT_MAX_GROUP);
    return DAOP_ERR_UNSUPPORTED;
  }
  cudaStream_t st = as_stream(stream);
  uint8_t* ws = static_cast<uint8_t*>(d_workspace);
  float* qkv = reinterpret_cast<float*>(ws);
  float* part = qkv + q_dim + 2 * kv_dim;
  const int group = n_heads / n_kv;
  uint16_t* o = reinterpret_cast<uint16_t*>(part + static_cast<int64_t>(n_kv) * 64 * group *
                                                       (2 + AT_HD));
  const int sms = sm_count();
  const size_t smem_qkv = static_cast<size_t>(d) * 2 + 33 * 4;
  DAOP_CUDA(cudaFuncSetAttribute(attn_qkv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_qkv)));
  attn_qkv_kernel<<<sms, AT_WARPS * 32, smem_qkv, st>>>(d_h, d_gamma, d_wqkv, d,
                                                        q_dim + 2 * kv_dim, eps, d_xa_out, qkv);
  DAOP_CHECK_LAUNCH("attn_qkv");
  // position splits: enough CTAs to cover the SMs, at least one tile each
  const int ctx = pos + 1;
  int splits = (sms + n_kv - 1) / n_kv;
  const int max_splits = (ctx + AT_TILE - 1) / AT_TILE;
  if (splits > max_splits) splits = max_splits;
  if (splits > 64) splits = 64;
  if (splits < 1) splits = 1;
  int per_split = (ctx + splits - 1) / splits;
  per_split = (per_split + AT_TILE - 1) / AT_TILE * AT_TILE;
  const int used = (ctx + per_split - 1) / per_split;
  AttnArgs a{qkv, d_k_cache, d_v_cache, n_heads, n_kv, max_seq, pos, splits, per_split,
             theta, 1.0f / sqrtf(static_cast<float>(AT_HD)), part};
  attn_decode_kernel<<<dim3(n_kv, used), AT_TILE, 0, st>>>(a);
  DAOP_CHECK_LAUNCH("attn_decode");
  attn_combine_kernel<<<n_heads, AT_HD, 0, st>>>(part, n_heads, n_kv, splits, used, o);
  DAOP_CHECK_LAUNCH("attn_combine");
  const size_t smem_o = static_cast<size_t>(q_dim) * 2;
  DAOP_CUDA(cudaFuncSetAttribute(attn_oproj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem_o)));
  attn_oproj_kernel<<<sms, AT_WARPS * 32, smem_o, st>>>(d_h, o, d_wo, d, q_dim, d_h_out);
  DAOP_CHECK_LAUNCH("attn_oproj");
  return DAOP_OK;
}
