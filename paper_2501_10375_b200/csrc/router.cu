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
  int prefetch_tiles;  // single-pass router: L2 prefetch distance in grid-strides (0: none)
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

// same, with shuffles limited to the P2 >= E lanes that hold experts
static __device__ __forceinline__ float lane_softmax_p2(float z, int lane, int E, int P2) {
  float m = lane < E ? z : -INFINITY;
  for (int o = P2 >> 1; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float e = lane < E ? expf(z - m) : 0.f;
  float s = e;
  for (int o = P2 >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return lane < E ? e / s : 0.f;
}

// GATE_IN_SMEM: gate rows staged in shared memory (they fit for d*2E*2 <= ~200 KB)
template <bool GATE_IN_SMEM>
__global__ void __launch_bounds__(kRouterWarps * 32)
    router_kernel(RouterArgs a) {
  pdl_prologue();  // (launched with launch_pdl)
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
    // pass 1: sum of squares (fp64, common.cuh rms_scale)
    double ss = 0.0;
    for (int c = lane; c < nchunk; c += 32) {
      const float4 u = reinterpret_cast<const float4*>(hrow)[2 * c];
      const float4 v = reinterpret_cast<const float4*>(hrow)[2 * c + 1];
      ss = sq_acc4(v, sq_acc4(u, ss));
    }
    ss = warp_sum(ss);
    const float r = rms_scale(ss, d, a.eps);
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
      bi = __shfl_sync(0xffffffffu, bi, 0);
      bv = __shfl_sync(0xffffffffu, bv, 0);
      if (bi >= E) {  // NaN scores never compare: first untaken id (topk_scan rule)
        bi = __ffs(__ballot_sync(0xffffffffu, !taken)) - 1;
        bv = __shfl_sync(0xffffffffu, p, bi);
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

// ---------------------------------------------------------------------------
// Tensor-core router (2E <= 16 gate rows, d % 256 == 0): the gate logits of
// 8 tokens are one m16n8k16 MMA chain -- gate rows are the M side (A, bf16
// from shared memory), the 8 tokens the N side (B, built in registers from
// this lane's own h values: lane holds token lane/4 at k = 2*(lane%4)+{0,1,8,9}
// of every 16-wide k-step, exactly the B-fragment layout, so x never touches
// shared memory).  16 warps split K; per-warp partials are summed in fixed
// warp order.  Two passes over the 8 rows of h: sum of squares (HBM), then
// x = bf16(h * r * gamma) + MMA (the rows are still in L2).  The kernel is
// HBM-bound on the h read + x write (16 + 8 KB per token at d = 4096).
constexpr int kMmaWarps = 16;
constexpr int kTokTile = 8;

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_x2(float h0, float h1, float r, uint32_t g2) {
  const float x0 = __fmul_rn(__fmul_rn(h0, r), bf16lo(g2));
  const float x1 = __fmul_rn(__fmul_rn(h1, r), bf16hi(g2));
  return static_cast<uint32_t>(f32_to_bf16_bits(x0)) |
         (static_cast<uint32_t>(f32_to_bf16_bits(x1)) << 16);
}

// L2 prefetch of a contiguous byte range (bulk, asynchronous, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)),
               "r"(bytes)
               : "memory");
}

// softmax / top-k / renormalisation / activation counter of token tt from
// its gate logits (zt own gate, zp next layer's), one expert per lane, shuffles
// over the P2 >= E lanes; ties -> lower id (topk_scan, moesim/_kernels.py:63-79)
__device__ __forceinline__ void token_finish(const RouterArgs& a, int64_t tt, int lane, float zt,
                                             float zp, int P2) {
  const int E = a.E;
  const float p = lane_softmax_p2(zt, lane, E, P2);
  if (lane < E) a.p_true[tt * E + lane] = p;
  if (a.wg_next) {
    const float ph = lane_softmax_p2(zp, lane, E, P2);
    if (lane < E) a.p_pred[tt * E + lane] = ph;
  }
  bool taken = lane >= E;
  int my_sel = -1;
  float my_p = 0.f, den = 0.f;
  for (int j = 0; j < a.k; ++j) {
    float bv = taken ? -INFINITY : p;
    int bi = taken ? 0x7fffffff : lane;
#pragma unroll
    for (int o = P2 >> 1; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    bi = __shfl_sync(0xffffffffu, bi, 0);
    bv = __shfl_sync(0xffffffffu, bv, 0);
    if (bi >= E) {  // NaN scores never compare: first untaken id
      bi = __ffs(__ballot_sync(0xffffffffu, !taken)) - 1;
      bv = __shfl_sync(0xffffffffu, p, bi);
    }
    den += bv;
    if (lane == j) {
      my_sel = bi;
      my_p = bv;
    }
    if (lane == bi) taken = true;
  }
  if (lane < a.k) {
    a.topk_idx[tt * a.k + lane] = my_sel;
    a.topk_w[tt * a.k + lane] = my_p / den;
    if (a.hist) atomicAdd(a.hist + (tt / a.tokens_per_seq) * a.hist_seq_stride + my_sel, 1);
  }
}

__global__ void __launch_bounds__(kMmaWarps * 32, 1) router_mma_kernel(RouterArgs a) {
  pdl_prologue();  // (launched with launch_pdl)
  extern __shared__ __align__(16) uint8_t smem[];
  const int d = a.d, E = a.E;
  const int rows = a.wg_next ? 2 * E : E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ld = d + 8;  // padded gate row (bf16): conflict-free fragment loads
  uint16_t* gs = reinterpret_cast<uint16_t*>(smem);                 // 16 x ld
  uint16_t* gam = gs + 16 * ld;                                       // d
  double* sspart = reinterpret_cast<double*>(gam + d);                // [2][kMmaWarps][8]
  float* zpart = reinterpret_cast<float*>(sspart + 2 * kMmaWarps * kTokTile);  // [2][kMmaWarps][16][8]

  for (int i = threadIdx.x; i < 16 * (d / 8); i += blockDim.x) {
    const int r = i / (d / 8), c = i - r * (d / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < E) v = reinterpret_cast<const uint4*>(a.wg + static_cast<size_t>(r) * d)[c];
    else if (r < rows) v = reinterpret_cast<const uint4*>(a.wg_next + static_cast<size_t>(r - E) * d)[c];
    *reinterpret_cast<uint4*>(gs + static_cast<size_t>(r) * ld + c * 8) = v;
  }
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x)
    reinterpret_cast<uint4*>(gam)[i] = reinterpret_cast<const uint4*>(a.gamma)[i];
  __syncthreads();

  const int g = lane >> 2, c2 = (lane & 3) * 2;  // fragment row / column pair
  int P2 = 1;
  while (P2 < E) P2 <<= 1;
  const int ksteps = d / (16 * kMmaWarps);
  const int k0w = warp * ksteps * 16;
  const int64_t ntiles = (a.T + kTokTile - 1) / kTokTile;
  // keep the h rows of the next PF tiles streaming into L2 (both passes then
  // read L2; the HBM stream runs ahead of the compute)
  constexpr int PF = 2;
  auto prefetch_tile = [&](int64_t tl) {
    if (tl >= ntiles) return;
    const int64_t t0 = tl * kTokTile;
    const int64_t n = (a.T - t0 < kTokTile ? a.T - t0 : kTokTile);
    for (int64_t q = 0; q < n; ++q) bulk_prefetch_l2(a.h + (t0 + q) * d, d * 4);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < PF; ++i) prefetch_tile(blockIdx.x + static_cast<int64_t>(i) * gridDim.x);
  // software pipeline over this CTA's tiles: the x/MMA pass of tile i and the
  // sum-of-squares pass of tile i+1 share one batch of loads and one barrier
  auto ss_partial = [&](double ssv) {  // sum over the 4 lanes of a token
    ssv += __shfl_xor_sync(0xffffffffu, ssv, 1);
    ssv += __shfl_xor_sync(0xffffffffu, ssv, 2);
    return ssv;
  };
  int buf = 0;
  {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kTokTile + g;
    double ss = 0.0;
    if (blockIdx.x < ntiles && t < a.T) {
      const float* hrow = a.h + t * d;
#pragma unroll 16
      for (int ks = 0; ks < ksteps; ++ks) {
        const int k = k0w + ks * 16 + c2;
        const float2 u = __ldg(reinterpret_cast<const float2*>(hrow + k));
        const float2 v = __ldg(reinterpret_cast<const float2*>(hrow + k + 8));
        ss = sq_acc(v.y, sq_acc(v.x, sq_acc(u.y, sq_acc(u.x, ss))));
      }
    }
    ss = ss_partial(ss);
    if ((lane & 3) == 0) sspart[warp * kTokTile + g] = ss;
    __syncthreads();
  }
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    if (threadIdx.x == 0) prefetch_tile(tile + static_cast<int64_t>(PF) * gridDim.x);
    const int64_t t = tile * kTokTile + g;  // this lane's token
    const bool live = t < a.T;
    const float* hrow = a.h + (live ? t : 0) * d;
    const int64_t t1 = t + static_cast<int64_t>(gridDim.x) * kTokTile;  // next tile, same lane
    const bool live1 = t1 < a.T;
    const float* hrow1 = a.h + (live1 ? t1 : 0) * d;
    const double* ssb = sspart + buf * kMmaWarps * kTokTile;
    double tot = 0.0;
    for (int w = 0; w < kMmaWarps; ++w) tot += ssb[w * kTokTile + g];
    const float r = rms_scale(tot, d, a.eps);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    double ss1 = 0.0;
    uint16_t* xrow = a.x_out ? a.x_out + (live ? t : 0) * d : nullptr;
    // batches of 4 k-steps: every h load of the batch (this tile's reload and
    // the next tile's first read) is issued before the x stores, which the
    // compiler cannot prove do not alias h
    for (int ks0 = 0; ks0 < ksteps; ks0 += 4) {
      float2 u[4], v[4], u1[4], v1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        u[i] = v[i] = u1[i] = v1[i] = make_float2(0.f, 0.f);
        if (ks0 + i < ksteps) {
          const int k = k0w + (ks0 + i) * 16 + c2;
          if (live) {
            u[i] = __ldg(reinterpret_cast<const float2*>(hrow + k));
            v[i] = __ldg(reinterpret_cast<const float2*>(hrow + k + 8));
          }
          if (live1) {
            u1[i] = __ldg(reinterpret_cast<const float2*>(hrow1 + k));
            v1[i] = __ldg(reinterpret_cast<const float2*>(hrow1 + k + 8));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ss1 = sq_acc(v1[i].y, sq_acc(v1[i].x, sq_acc(u1[i].y, sq_acc(u1[i].x, ss1))));
        if (ks0 + i < ksteps) {
          const int k = k0w + (ks0 + i) * 16 + c2;
          const uint32_t b0 = pack_x2(u[i].x, u[i].y, r, *reinterpret_cast<const uint32_t*>(gam + k));
          const uint32_t b1 =
              pack_x2(v[i].x, v[i].y, r, *reinterpret_cast<const uint32_t*>(gam + k + 8));
          if (live && xrow) {
            *reinterpret_cast<uint32_t*>(xrow + k) = b0;
            *reinterpret_cast<uint32_t*>(xrow + k + 8) = b1;
          }
          uint32_t af[4];
          af[0] = *reinterpret_cast<const uint32_t*>(gs + g * ld + k);
          af[1] = *reinterpret_cast<const uint32_t*>(gs + (g + 8) * ld + k);
          af[2] = *reinterpret_cast<const uint32_t*>(gs + g * ld + k + 8);
          af[3] = *reinterpret_cast<const uint32_t*>(gs + (g + 8) * ld + k + 8);
          mma_bf16_16816(acc, af, b0, b1);
        }
      }
    }
    ss1 = ss_partial(ss1);
    if ((lane & 3) == 0) sspart[(buf ^ 1) * kMmaWarps * kTokTile + warp * kTokTile + g] = ss1;
    // D fragment: gate rows g, g+8 x tokens c2, c2+1
    float* zb = zpart + buf * kMmaWarps * 16 * kTokTile + warp * 16 * kTokTile;
    zb[g * kTokTile + c2] = acc[0];
    zb[g * kTokTile + c2 + 1] = acc[1];
    zb[(g + 8) * kTokTile + c2] = acc[2];
    zb[(g + 8) * kTokTile + c2 + 1] = acc[3];
    __syncthreads();
    // token phase: warp w < 8 finishes token w of the tile (one expert per lane)
    if (warp < kTokTile) {
      const int64_t tt = tile * kTokTile + warp;
      if (tt < a.T) {
        const float* z0 = zpart + buf * kMmaWarps * 16 * kTokTile;
        float zt = 0.f, zp = 0.f;
        if (lane < E) {
          for (int w = 0; w < kMmaWarps; ++w) {
            zt += z0[(w * 16 + lane) * kTokTile + warp];
            if (a.wg_next) zp += z0[(w * 16 + E + lane) * kTokTile + warp];
          }
        }
        token_finish(a, tt, lane, zt, zp, P2);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Single-pass tensor-core router (d = 256 * KS, KS <= 16: every Mixtral-8x7B
// sized model).  Same tile / fragment scheme as router_mma_kernel, but each
// lane keeps its token's h slice (KS x 4 floats) in registers from the one
// read that feeds both the sum of squares and the x / MMA pass: h crosses
// HBM once (L2 prefetch of the tiles PF grid-strides ahead) and L2 once,
// instead of L2 twice.  Two CTA barriers per tile: the RMS partials, then
// the logit partials; warps 8..15 start the next tile while 0..7 finish the
// tokens of this one.
template <int KS>
__global__ void __launch_bounds__(kMmaWarps * 32, 1) router_mma1_kernel(RouterArgs a) {
  pdl_prologue();  // (launched with launch_pdl)
  extern __shared__ __align__(16) uint8_t smem[];
  const int d = a.d, E = a.E;
  const int rows = a.wg_next ? 2 * E : E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ld = d + 8;
  uint16_t* gs = reinterpret_cast<uint16_t*>(smem);                  // 16 x ld
  uint16_t* gam = gs + 16 * ld;                                        // d
  double* sspart = reinterpret_cast<double*>(gam + d);                 // [kMmaWarps][8]
  float* zpart = reinterpret_cast<float*>(sspart + kMmaWarps * kTokTile);  // [kMmaWarps][16][8]
  for (int i = threadIdx.x; i < 16 * (d / 8); i += blockDim.x) {
    const int r = i / (d / 8), c = i - r * (d / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < E) v = reinterpret_cast<const uint4*>(a.wg + static_cast<size_t>(r) * d)[c];
    else if (r < rows) v = reinterpret_cast<const uint4*>(a.wg_next + static_cast<size_t>(r - E) * d)[c];
    *reinterpret_cast<uint4*>(gs + static_cast<size_t>(r) * ld + c * 8) = v;
  }
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x)
    reinterpret_cast<uint4*>(gam)[i] = reinterpret_cast<const uint4*>(a.gamma)[i];
  __syncthreads();

  const int g = lane >> 2, c2 = (lane & 3) * 2;
  int P2 = 1;
  while (P2 < E) P2 <<= 1;
  const int k0w = warp * KS * 16;
  const int64_t ntiles = (a.T + kTokTile - 1) / kTokTile;
  const int PF = a.prefetch_tiles;
  auto prefetch_tile = [&](int64_t tl) {
    if (PF <= 0 || tl >= ntiles) return;
    const int64_t t0 = tl * kTokTile;
    const int64_t n = (a.T - t0 < kTokTile ? a.T - t0 : kTokTile);
    bulk_prefetch_l2(a.h + t0 * d, static_cast<uint32_t>(n * d * 4));  // rows are contiguous
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < PF; ++i) prefetch_tile(blockIdx.x + static_cast<int64_t>(i) * gridDim.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (threadIdx.x == 0) prefetch_tile(tile + static_cast<int64_t>(PF) * gridDim.x);
    const int64_t t = tile * kTokTile + g;
    const bool live = t < a.T;
    const float* hrow = a.h + (live ? t : 0) * d;
    float2 u[KS], v[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = k0w + ks * 16 + c2;
      u[ks] = live ? __ldg(reinterpret_cast<const float2*>(hrow + k)) : make_float2(0.f, 0.f);
      v[ks] = live ? __ldg(reinterpret_cast<const float2*>(hrow + k + 8)) : make_float2(0.f, 0.f);
    }
    double ss = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
      ss = sq_acc(v[ks].y, sq_acc(v[ks].x, sq_acc(u[ks].y, sq_acc(u[ks].x, ss))));
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    if ((lane & 3) == 0) sspart[warp * kTokTile + g] = ss;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < kMmaWarps; ++w) tot += sspart[w * kTokTile + g];
    const float r = rms_scale(tot, d, a.eps);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    uint16_t* xrow = a.x_out ? a.x_out + (live ? t : 0) * d : nullptr;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = k0w + ks * 16 + c2;
      const uint32_t b0 = pack_x2(u[ks].x, u[ks].y, r, *reinterpret_cast<const uint32_t*>(gam + k));
      const uint32_t b1 = pack_x2(v[ks].x, v[ks].y, r, *reinterpret_cast<const uint32_t*>(gam + k + 8));
      if (live && xrow) {
        *reinterpret_cast<uint32_t*>(xrow + k) = b0;
        *reinterpret_cast<uint32_t*>(xrow + k + 8) = b1;
      }
      uint32_t af[4];
      af[0] = *reinterpret_cast<const uint32_t*>(gs + g * ld + k);
      af[1] = *reinterpret_cast<const uint32_t*>(gs + (g + 8) * ld + k);
      af[2] = *reinterpret_cast<const uint32_t*>(gs + g * ld + k + 8);
      af[3] = *reinterpret_cast<const uint32_t*>(gs + (g + 8) * ld + k + 8);
      mma_bf16_16816(acc, af, b0, b1);
    }
    float* zb = zpart + warp * 16 * kTokTile;
    zb[g * kTokTile + c2] = acc[0];
    zb[g * kTokTile + c2 + 1] = acc[1];
    zb[(g + 8) * kTokTile + c2] = acc[2];
    zb[(g + 8) * kTokTile + c2 + 1] = acc[3];
    __syncthreads();
    if (warp < kTokTile) {
      const int64_t tt = tile * kTokTile + warp;
      if (tt < a.T) {
        float zt = 0.f, zp = 0.f;
        if (lane < E) {
          for (int w = 0; w < kMmaWarps; ++w) {
            zt += zpart[(w * 16 + lane) * kTokTile + warp];
            if (a.wg_next) zp += zpart[(w * 16 + E + lane) * kTokTile + warp];
          }
        }
        token_finish(a, tt, lane, zt, zp, P2);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Bulk-copy router (d = 256 * KS, KS in {8, 16}; 2E <= 16): the default for
// prompt-sized T.  The register-resident kernel above issues a tile's h loads
// only after the previous tile's logits are done, so HBM idles through every
// RMS / MMA / top-k phase (3.0 TB/s).  Here thread 0 streams 4-token tiles
// (4 contiguous rows, one cp.async.bulk of 4 * d * 4 B, L2 evict_first) into
// a ring of `stages` shared-memory stages (3 x 64 KB at d = 4096; a stage is
// refilled right after the barrier that ends its tile), so two tiles are in
// flight while the 16 warps work on the third.  (A dedicated producer warp
// would cap the 17-warp CTA at 96 registers and spill.)  The gate rows do not
// live in shared memory: warp w owns the d-slice [w S, (w + 1) S), S = 16 KS,
// and keeps its A fragments (rows g, g + 8 of the slice) in registers.
// Per tile, two CTA barriers:
//   pass 1  warps 0..14: fp64 sums of squares, float4s lane-strided over the
//           whole row (doubles assembled with integer ops: F2F.F64 is issued
//           through MIO and was the pass's bottleneck); a transposed butterfly
//           leaves token (lane >> 3)'s sum in lanes 0, 8, 16, 24; the last
//           warp to arrive (shared-memory counter) turns the 15 partials into
//           r in fixed warp order.  Warp 15 meanwhile finishes the PREVIOUS
//           tile's 4 tokens (lane = token * 8 + expert: segmented softmax of
//           both gates, top-k, renormalisation, counter).
//   -- barrier A --
//   pass 2  every warp: x = bf16(h * r * gamma) of its slice, in place in the
//           stage (row tok shifted by tok * 16 B) and to x_out (8-byte
//           coalesced stores); the slice's m16n8k16 chain with B fragments by
//           ldmatrix.x4 (tokens 0..3 = columns 0..3; rows 4..7 repeat 0..3
//           and their columns are discarded); partial logits -> zpart
//   -- barrier B --  stage refill
// The logits are the same MMA chains over the same 16-column k-steps as
// router_mma1_kernel<KS>, summed over warps in the same order.
// Measured (profiles/r02/stream_kernels.json, ncu_router_bulk.json): 32,768 tokens x d = 4096 in
// ~164 us = 4.9 TB/s of algorithmic bytes (register-resident: 269 us).
constexpr int kTmaTok = 4;
constexpr int kPass1Warps = kMmaWarps - 1;

// |v| as a double built with integer ops (the ALU pipe) instead of
// F2F.F64.F32 (MIO-issued, the pass-1 bottleneck): exact for normal floats;
// zeros / subnormals become values below 2^-126 whose squares (< 2^-252)
// vanish in any fp64 sum that matters and underflow the f32 mean otherwise;
// Inf / NaN become finite values >= 2^128 (squares >= 2^256, an f32 mean of
// Inf -> r = 0 exactly as for Inf); NaN is restored by the caller from `mx`.
__device__ __forceinline__ double abs_f32_as_f64(float v, uint32_t& mx) {
  const uint32_t t = __float_as_uint(v) << 1;  // |v| bits, shifted left once
  mx = max(mx, t);
  return __hiloint2double((t >> 4) + 0x38000000u, __float_as_uint(v) << 29);
}

__device__ __forceinline__ double sq_acc4_int(float4 v, double a, uint32_t& mx) {
  double x = abs_f32_as_f64(v.x, mx);
  a = fma(x, x, a);
  x = abs_f32_as_f64(v.y, mx);
  a = fma(x, x, a);
  x = abs_f32_as_f64(v.z, mx);
  a = fma(x, x, a);
  x = abs_f32_as_f64(v.w, mx);
  return fma(x, x, a);
}

// finish 4 tokens of a tile in one warp: lane = tok * 8 + e (E <= 8)
__device__ __forceinline__ void tile_finish(const RouterArgs& a, int64_t t0, int n, int lane,
                                            const float* zpart) {
  const int E = a.E, tok = lane >> 3, e = lane & 7;
  const bool ex = e < E;
  float zt = 0.f, zp = 0.f;
  if (ex) {
#pragma unroll
    for (int w = 0; w < kMmaWarps; ++w) {
      zt += zpart[(w * 16 + e) * kTmaTok + tok];
      if (a.wg_next) zp += zpart[(w * 16 + E + e) * kTmaTok + tok];
    }
  }
  // segmented softmax over the 8 lanes of the token (== lane_softmax_p2: the
  // extra lanes contribute -inf to the max and +0 to the sum)
  float m = ex ? zt : -INFINITY, mp = ex ? zp : -INFINITY;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    mp = fmaxf(mp, __shfl_xor_sync(0xffffffffu, mp, o));
  }
  const float et = ex ? expf(zt - m) : 0.f, ep = ex ? expf(zp - mp) : 0.f;
  float st = et, sp = ep;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    st += __shfl_xor_sync(0xffffffffu, st, o);
    sp += __shfl_xor_sync(0xffffffffu, sp, o);
  }
  const float p = ex ? et / st : 0.f;
  const bool live = tok < n;
  const int64_t tt = t0 + tok;
  if (live && ex) {
    a.p_true[tt * E + e] = p;
    if (a.wg_next) a.p_pred[tt * E + e] = ep / sp;
  }
  const int seg = lane & ~7;
  bool taken = !ex;
  int my_sel = -1;
  float my_p = 0.f, den = 0.f;
  for (int j = 0; j < a.k; ++j) {
    float bv = taken ? -INFINITY : p;
    int bi = taken ? 0x7fffffff : e;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    bi = __shfl_sync(0xffffffffu, bi, seg);
    bv = __shfl_sync(0xffffffffu, bv, seg);
    if (bi >= E) {  // NaN scores never compare: first untaken id (topk_scan rule)
      const unsigned free_ = (__ballot_sync(0xffffffffu, !taken) >> seg) & 0xffu;
      bi = __ffs(free_) - 1;
      bv = __shfl_sync(0xffffffffu, p, seg + bi);
    }
    den += bv;
    if (e == j) {
      my_sel = bi;
      my_p = bv;
    }
    if (e == bi) taken = true;
  }
  if (live && e < a.k) {
    a.topk_idx[tt * a.k + e] = my_sel;
    a.topk_w[tt * a.k + e] = my_p / den;
    if (a.hist) atomicAdd(a.hist + (tt / a.tokens_per_seq) * a.hist_seq_stride + my_sel, 1);
  }
}

template <int KS>
__global__ void __launch_bounds__(kMmaWarps * 32, 1) router_tma_kernel(RouterArgs a, int stages) {
  pdl_prologue();  // (launched with launch_pdl)
  constexpr int TOK = kTmaTok;
  constexpr int S = KS * 16;                   // d-slice per warp
  constexpr int NV4 = KS / 8;                  // float4s per lane per token row of the slice
  constexpr int NV4ROW = KS * 64;              // float4s per row (d / 4)
  constexpr int P1 = kPass1Warps * 32;         // pass-1 lanes
  constexpr int P1FULL = NV4ROW / P1, P1REM = NV4ROW % P1;
  extern __shared__ __align__(128) uint8_t smem[];
  const int d = a.d, E = a.E;
  const int rows = a.wg_next ? 2 * E : E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t stage_bytes = static_cast<uint32_t>(TOK) * d * 4;
  uint8_t* ring = smem;
  double* sspart = reinterpret_cast<double*>(smem + static_cast<size_t>(stages) * stage_bytes);
  float* zpart = reinterpret_cast<float*>(sspart + kMmaWarps * TOK);  // [warp][16 rows][TOK]
  float* rs = zpart + kMmaWarps * 16 * TOK;                           // [TOK]
  unsigned* arrived = reinterpret_cast<unsigned*>(rs + TOK);
  uint64_t* full = reinterpret_cast<uint64_t*>(rs + 8);
  const int64_t ntiles = (a.T + TOK - 1) / TOK;
  uint64_t pol = 0;
  // thread 0 issues tile i's copy into stage i % stages: the first `stages`
  // tiles here, tile i + stages right after the barrier that ends tile i
  auto issue = [&](int64_t tile, int s) {
    if (tile >= ntiles) return;
    const int64_t t0 = tile * TOK;
    const int64_t n = a.T - t0 < TOK ? a.T - t0 : TOK;
    const uint32_t bytes = static_cast<uint32_t>(n * d * 4);
    mbar_arrive_expect_tx(&full[s], bytes);
    bulk_g2s(ring + static_cast<size_t>(s) * stage_bytes, a.h + t0 * d, bytes, &full[s], pol);
  };
  if (threadIdx.x == 0) {
    pol = l2_evict_first_policy();
    *arrived = 0;
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    for (int s = 0; s < stages; ++s) issue(blockIdx.x + static_cast<int64_t>(s) * gridDim.x, s);
  }
  __syncthreads();

  const int g = lane >> 2, c = lane & 3, c2 = c * 2;
  const int base = warp * S;
  uint32_t af[KS][4];
  {
    const uint16_t* r0 = g < E ? a.wg + static_cast<size_t>(g) * d
                               : (g < rows ? a.wg_next + static_cast<size_t>(g - E) * d : nullptr);
    const int g8 = g + 8;
    const uint16_t* r1 = g8 < E ? a.wg + static_cast<size_t>(g8) * d
                                : (g8 < rows ? a.wg_next + static_cast<size_t>(g8 - E) * d : nullptr);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = base + ks * 16 + c2;
      af[ks][0] = r0 ? __ldg(reinterpret_cast<const uint32_t*>(r0 + k)) : 0u;
      af[ks][1] = r1 ? __ldg(reinterpret_cast<const uint32_t*>(r1 + k)) : 0u;
      af[ks][2] = r0 ? __ldg(reinterpret_cast<const uint32_t*>(r0 + k + 8)) : 0u;
      af[ks][3] = r1 ? __ldg(reinterpret_cast<const uint32_t*>(r1 + k + 8)) : 0u;
    }
  }
  uint2 gm[NV4];
#pragma unroll
  for (int j = 0; j < NV4; ++j)
    gm[j] = *reinterpret_cast<const uint2*>(a.gamma + base + j * 128 + lane * 4);
  const bool hi16 = lane & 16, hi8 = lane & 8;
  const int p1 = warp * 32 + lane;                    // pass-1 lane id (warps 0..14)
  const double inv_d = 1.0 / static_cast<double>(d);  // d = 2^11 / 2^12: exact
  int64_t prev_t0 = -1;
  int prev_n = 0;
  int s = 0;
  uint32_t phase = 0;  // parity of stage s's current fill
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint8_t* st = ring + static_cast<size_t>(s) * stage_bytes;
    const int64_t t0 = tile * TOK;
    const int n = static_cast<int>(a.T - t0 < TOK ? a.T - t0 : TOK);
    if (warp < kPass1Warps) {
      // pass 1: fp64 sums of squares of the 4 rows, lane-strided float4s
      mbar_wait(&full[s], phase);
      double ss[TOK];
#pragma unroll
      for (int tok = 0; tok < TOK; ++tok) {
        const float4* hrow = reinterpret_cast<const float4*>(st) + tok * NV4ROW + p1;
        double v = 0.0;
        uint32_t mx = 0;
#pragma unroll
        for (int j = 0; j < P1FULL; ++j) v = sq_acc4_int(hrow[j * P1], v, mx);
        if (p1 < P1REM) v = sq_acc4_int(hrow[P1FULL * P1], v, mx);
        ss[tok] = mx > 0xff000000u ? __longlong_as_double(0x7ff8000000000000ll) : v;  // NaN in
      }
      const double s0 = __shfl_xor_sync(0xffffffffu, hi16 ? ss[0] : ss[2], 16);
      const double s1 = __shfl_xor_sync(0xffffffffu, hi16 ? ss[1] : ss[3], 16);
      const double k0 = (hi16 ? ss[2] : ss[0]) + s0;
      const double k1 = (hi16 ? ss[3] : ss[1]) + s1;
      const double s2 = __shfl_xor_sync(0xffffffffu, hi8 ? k0 : k1, 8);
      double v = (hi8 ? k1 : k0) + s2;
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if ((lane & 7) == 0) sspart[warp * TOK + (lane >> 3)] = v;
      // the last pass-1 warp turns the partials into r (fixed warp order)
      __threadfence_block();
      __syncwarp();
      unsigned last = 0;
      if (lane == 0) last = atomicAdd(arrived, 1u) == kPass1Warps - 1;
      if (__shfl_sync(0xffffffffu, last, 0)) {
        __threadfence_block();
        if (lane < TOK) {
          double tot = 0.0;
#pragma unroll
          for (int w = 0; w < kPass1Warps; ++w) tot += sspart[w * TOK + lane];
          const float ms = static_cast<float>(tot * inv_d);
          rs[lane] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, a.eps)));
        }
        if (lane == 0) *arrived = 0;
      }
    } else {
      if (prev_t0 >= 0) tile_finish(a, prev_t0, prev_n, lane, zpart);
      mbar_wait(&full[s], phase);
    }
    __syncthreads();  // A
    // pass 2: x in place (row tok of the slice shifted by tok * 16 B) and to
    // x_out, then the slice's MMA chain
#pragma unroll
    for (int tok = 0; tok < TOK; ++tok) {
      const float r = rs[tok];
      const float* hrow = reinterpret_cast<const float*>(st) + static_cast<size_t>(tok) * d + base;
      float4 hv[NV4];
#pragma unroll
      for (int j = 0; j < NV4; ++j) hv[j] = *reinterpret_cast<const float4*>(hrow + j * 128 + lane * 4);
      __syncwarp();
      uint8_t* xs = st + static_cast<size_t>(tok) * d * 4 + static_cast<size_t>(base) * 4 + tok * 16;
#pragma unroll
      for (int j = 0; j < NV4; ++j) {
        uint2 xw;
        xw.x = cvt_bf16x2(__fmul_rn(__fmul_rn(hv[j].x, r), bf16lo(gm[j].x)),
                          __fmul_rn(__fmul_rn(hv[j].y, r), bf16hi(gm[j].x)));
        xw.y = cvt_bf16x2(__fmul_rn(__fmul_rn(hv[j].z, r), bf16lo(gm[j].y)),
                          __fmul_rn(__fmul_rn(hv[j].w, r), bf16hi(gm[j].y)));
        *reinterpret_cast<uint2*>(xs + (j * 128 + lane * 4) * 2) = xw;
        if (a.x_out && tok < n)
          *reinterpret_cast<uint2*>(a.x_out + (t0 + tok) * d + base + j * 128 + lane * 4) = xw;
      }
    }
    __syncwarp();
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    {
      // ldmatrix row = token (lane & 3; rows 4..7 repeat 0..3, their columns
      // are discarded), matrix = 8-column quarter of the k-step pair
      const int rt = lane & 3, q = lane >> 3;
      const uint8_t* xr = st + static_cast<size_t>(rt) * d * 4 + static_cast<size_t>(base) * 4 +
                          rt * 16 + q * 16;
#pragma unroll
      for (int pp = 0; pp < KS / 2; ++pp) {
          const uint4 b = ldmatrix_x4(xr + pp * 64);
        mma_bf16_16816(acc, af[2 * pp], b.x, b.y);
        mma_bf16_16816(acc, af[2 * pp + 1], b.z, b.w);
      }
    }
    fence_proxy_async();  // this warp's generic smem traffic before the stage's refill
    float* zb = zpart + warp * 16 * TOK;
    if (c2 < TOK) {
      zb[g * TOK + c2] = acc[0];
      zb[g * TOK + c2 + 1] = acc[1];
      zb[(g + 8) * TOK + c2] = acc[2];
      zb[(g + 8) * TOK + c2 + 1] = acc[3];
    }
    __syncthreads();  // B
    if (threadIdx.x == 0) issue(tile + static_cast<int64_t>(stages) * gridDim.x, s);
    prev_t0 = t0;
    prev_n = n;
    if (++s == stages) {
      s = 0;
      phase ^= 1u;
    }
  }
  if (warp == kMmaWarps - 1 && prev_t0 >= 0) tile_finish(a, prev_t0, prev_n, lane, zpart);
}

// ---------------------------------------------------------------------------
// Decode-sized batches (T <= 128): one CTA per token, 16 warps splitting d.
// The tensor-core router above amortises its 128 KB gate staging over many
// 8-token tiles; with a handful of tokens it would run a few CTAs through
// long dependent chains.  Here every token gets an SM: RMSNorm by a block
// reduction, the 2E gate dot products as per-warp partials reduced in fixed
// warp order, then the same softmax / top-k / renormalisation / counter as
// router_kernel (lane-parallel, ties -> lower id).
constexpr int kSmallWarps = 16;

__global__ void __launch_bounds__(kSmallWarps * 32, 1) router_small_kernel(RouterArgs a) {
  pdl_prologue();  // (launched with launch_pdl)
  const int d = a.d, E = a.E, k = a.k;
  const int rows = a.wg_next ? 2 * E : E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  const int64_t t = blockIdx.x;
  __shared__ double red[kSmallWarps];
  __shared__ float part[kSmallWarps][kMaxGateRows];
  const float* hrow = a.h + t * d;
  const int n8 = d / 8;  // 8-element chunks, thread-strided
  auto gate_chunk = [&](int q, int c) {
    const uint16_t* grow = q < E ? a.wg + static_cast<size_t>(q) * d
                                 : a.wg_next + static_cast<size_t>(q - E) * d;
    return ldg_nc_v4(reinterpret_cast<const uint4*>(grow) + c);
  };
  // the thread's first chunk of h, gamma and the first 16 gate rows are all
  // requested up front: their L2 round trip overlaps the RMS reduction
  const bool has0 = tid < n8;
  float4 u0 = make_float4(0.f, 0.f, 0.f, 0.f), v0 = u0;
  uint4 gm0 = make_uint4(0, 0, 0, 0);
  uint4 gv0[16];
  if (has0) {
    u0 = reinterpret_cast<const float4*>(hrow)[2 * tid];
    v0 = reinterpret_cast<const float4*>(hrow)[2 * tid + 1];
    gm0 = reinterpret_cast<const uint4*>(a.gamma)[tid];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) gv0[i] = has0 && i < rows ? gate_chunk(i, tid) : make_uint4(0, 0, 0, 0);
  double ss = has0 ? sq_acc4(v0, sq_acc4(u0, 0.0)) : 0.0;
  for (int c = tid + blockDim.x; c < n8; c += blockDim.x) {
    const float4 u = reinterpret_cast<const float4*>(hrow)[2 * c];
    const float4 v = reinterpret_cast<const float4*>(hrow)[2 * c + 1];
    ss = sq_acc4(v, sq_acc4(u, ss));
  }
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < kSmallWarps; ++w) tot += red[w];
  const float r = rms_scale(tot, d, a.eps);
  float acc[kMaxGateRows];
#pragma unroll
  for (int q = 0; q < kMaxGateRows; ++q) acc[q] = 0.f;
  auto x_of = [&](int c, float4 u, float4 v, uint4 gm) {
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
    return x8;
  };
  // rows 16..31 (E = 16 with the next-layer gate) of one chunk, batched
  auto rows_hi = [&](int c, uint4 x8) {
    if (rows > 16) {
      uint4 gv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) gv[i] = 16 + i < rows ? gate_chunk(16 + i, c) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (16 + i < rows) acc[16 + i] = dot8(x8, gv[i], acc[16 + i]);
    }
  };
  if (has0) {
    const uint4 x8 = x_of(tid, u0, v0, gm0);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < rows) acc[i] = dot8(x8, gv0[i], acc[i]);
    rows_hi(tid, x8);
  }
  for (int c = tid + blockDim.x; c < n8; c += blockDim.x) {
    const uint4 x8 = x_of(c, reinterpret_cast<const float4*>(hrow)[2 * c],
                          reinterpret_cast<const float4*>(hrow)[2 * c + 1],
                          reinterpret_cast<const uint4*>(a.gamma)[c]);
    uint4 gv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) gv[i] = i < rows ? gate_chunk(i, c) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < rows) acc[i] = dot8(x8, gv[i], acc[i]);
    rows_hi(c, x8);
  }
#pragma unroll
  for (int q = 0; q < kMaxGateRows; ++q)
    if (q < rows) {
      const float z = warp_sum(acc[q]);
      if (lane == 0) part[warp][q] = z;
    }
  __syncthreads();
  if (warp != 0) return;
  float zt = 0.f, zp = 0.f;
  if (lane < E)
    for (int w = 0; w < kSmallWarps; ++w) {
      zt += part[w][lane];
      if (a.wg_next) zp += part[w][E + lane];
    }
  const float p = lane_softmax(zt, lane, E);
  if (lane < E) a.p_true[t * E + lane] = p;
  if (a.wg_next) {
    const float ph = lane_softmax(zp, lane, E);
    if (lane < E) a.p_pred[t * E + lane] = ph;
  }
  bool taken = lane >= E;
  int my_sel = -1;
  float my_p = 0.f, den = 0.f;
  for (int j = 0; j < k; ++j) {
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
    bi = __shfl_sync(0xffffffffu, bi, 0);
    bv = __shfl_sync(0xffffffffu, bv, 0);
    if (bi >= E) {  // NaN scores never compare: first untaken id (topk_scan rule)
      bi = __ffs(__ballot_sync(0xffffffffu, !taken)) - 1;
      bv = __shfl_sync(0xffffffffu, p, bi);
    }
    den += bv;
    if (lane == j) {
      my_sel = bi;
      my_p = bv;
    }
    if (lane == bi) taken = true;
  }
  if (lane < k) {
    a.topk_idx[t * k + lane] = my_sel;
    a.topk_w[t * k + lane] = my_p / den;
    if (a.hist) atomicAdd(a.hist + (t / a.tokens_per_seq) * a.hist_seq_stride + my_sel, 1);
  }
}

}  // namespace daop

using namespace daop;

// tuning switch (daop_set_router_mode): 1 = single-pass router where it applies
static int g_router_single_pass = 1;
static int g_router_prefetch = 1;
static int g_router_tma = 1;
static int g_router_small_bulk = 0;  // tuning: bulk router also for 8 <= T <= 128

// bit 0: single pass; bit 2: bulk-copy router OFF; bit 3: bulk router for
// 8 <= T <= 128 too (instead of a CTA per token); bits 4..7: + 1 = L2
// prefetch distance of the single-pass kernel in grid-strides (0 in those
// bits keeps the current distance)
extern "C" int daop_set_router_mode(int32_t mode) {
  g_router_single_pass = mode & 1;
  g_router_tma = (mode & 4) ? 0 : 1;
  g_router_small_bulk = (mode >> 3) & 1;
  if ((mode >> 4) & 15) g_router_prefetch = ((mode >> 4) & 15) - 1;
  return DAOP_OK;
}

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
               topk_idx, topk_w, hist, tokens_per_seq, hist_seq_stride, g_router_prefetch};
  const int rows = wg_next ? 2 * E : E;
  const int ks_small = d % (16 * kMmaWarps) == 0 ? d / (16 * kMmaWarps) : 0;
  const bool tma_ok = rows <= 16 && E <= 8 && g_router_single_pass && g_router_tma &&
                      (ks_small == 8 || ks_small == 16);
  if (T <= 128 && d % 8 == 0 && !(g_router_small_bulk && tma_ok && T >= 8)) {
    // decode-sized batch: a CTA per token
    DAOP_CUDA(launch_pdl(router_small_kernel, dim3(static_cast<int>(T)), dim3(kSmallWarps * 32), 0, as_stream(st), a));
    DAOP_CHECK_LAUNCH("router_small");
    return DAOP_OK;
  }
  const int ks1 = d % (16 * kMmaWarps) == 0 ? d / (16 * kMmaWarps) : 0;
  // bulk-copy router: d = 256 * KS with KS in {8, 16}, E <= 8 (one finisher warp)
  if (rows <= 16 && E <= 8 && g_router_single_pass && g_router_tma && (ks1 == 8 || ks1 == 16)) {
    const size_t stage = static_cast<size_t>(kTmaTok) * d * 4;
    const size_t fixed = kMmaWarps * kTmaTok * 8 + kMmaWarps * 16 * kTmaTok * 4 + 8 * 4 + 8 * 8;
    int stages = static_cast<int>((232448 - fixed) / stage);
    if (stages > 6) stages = 6;
    const size_t smem = stages * stage + fixed;
    const int64_t ntiles = (T + kTmaTok - 1) / kTmaTok;
    const int blocks = static_cast<int>(ntiles < sm_count() ? ntiles : sm_count());
    auto launch = [&](auto kern) {
      DAOP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      DAOP_CUDA(launch_pdl(kern, dim3(blocks), dim3(kMmaWarps * 32), smem, as_stream(st), a, stages));
      return DAOP_OK;
    };
    const int rc = ks1 == 8 ? launch(router_tma_kernel<8>) : launch(router_tma_kernel<16>);
    if (rc) return rc;
    DAOP_CHECK_LAUNCH("router_tma");
    return DAOP_OK;
  }
  // single-pass router: d = 256 * KS with KS in {4, 8, 12, 16} (h slice in registers)
  if (rows <= 16 && g_router_single_pass && (ks1 == 4 || ks1 == 8 || ks1 == 12 || ks1 == 16)) {
    const size_t smem1 = static_cast<size_t>(16) * (d + 8) * 2 + static_cast<size_t>(d) * 2 +
                         kMmaWarps * kTokTile * 8 + kMmaWarps * 16 * kTokTile * 4;
    const int64_t ntiles = (T + kTokTile - 1) / kTokTile;
    const int blocks = static_cast<int>(ntiles < sm_count() ? ntiles : sm_count());
    auto launch1 = [&](auto kern) {
      DAOP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem1)));
      DAOP_CUDA(launch_pdl(kern, dim3(blocks), dim3(kMmaWarps * 32), smem1, as_stream(st), a));
      return DAOP_OK;
    };
    int rc = ks1 == 4 ? launch1(router_mma1_kernel<4>) : ks1 == 8 ? launch1(router_mma1_kernel<8>)
             : ks1 == 12 ? launch1(router_mma1_kernel<12>) : launch1(router_mma1_kernel<16>);
    if (rc) return rc;
    DAOP_CHECK_LAUNCH("router_single_pass");
    return DAOP_OK;
  }
  const size_t smem_mma = static_cast<size_t>(16) * (d + 8) * 2 + static_cast<size_t>(d) * 2 +
                          2 * kMmaWarps * kTokTile * 8 + 2 * kMmaWarps * 16 * kTokTile * 4;
  if (rows <= 16 && d % (16 * kMmaWarps) == 0 && smem_mma <= 232448) {
    const int64_t ntiles = (T + kTokTile - 1) / kTokTile;
    const int blocks = static_cast<int>(ntiles < sm_count() ? ntiles : sm_count());
    DAOP_CUDA(cudaFuncSetAttribute(router_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem_mma)));
    DAOP_CUDA(launch_pdl(router_mma_kernel, dim3(blocks), dim3(kMmaWarps * 32), smem_mma, as_stream(st), a));
    DAOP_CHECK_LAUNCH("router");
    return DAOP_OK;
  }
  const size_t smem = static_cast<size_t>(rows) * d * 2;
  int64_t blocks = (T + kRouterWarps - 1) / kRouterWarps;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 2;
  if (smem <= 100 * 1024) {
    if (blocks > cap) blocks = cap;
    DAOP_CUDA(cudaFuncSetAttribute(router_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    DAOP_CUDA(launch_pdl(router_kernel<true>, dim3(static_cast<int>(blocks)), dim3(kRouterWarps * 32), smem, as_stream(st), a));
  } else if (smem <= 200 * 1024 && T >= 4096) {
    const int64_t cap1 = sm_count();
    if (blocks > cap1) blocks = cap1;
    DAOP_CUDA(cudaFuncSetAttribute(router_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    DAOP_CUDA(launch_pdl(router_kernel<true>, dim3(static_cast<int>(blocks)), dim3(kRouterWarps * 32), smem, as_stream(st), a));
  } else {
    if (blocks > cap * 4) blocks = cap * 4;
    DAOP_CUDA(launch_pdl(router_kernel<false>, dim3(static_cast<int>(blocks)), dim3(kRouterWarps * 32), 0, as_stream(st), a));
  }
  DAOP_CHECK_LAUNCH("router");
  return DAOP_OK;
}
