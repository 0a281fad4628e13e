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
// Three launches, each HBM-bound on what it streams:
//   attn_qkv_kernel      warp-per-row GEMV over Wqkv (50 MB at 8x7B); every CTA first
//                        prefetches its rows into L2, then computes the RMSNorm
//   attn_decode_kernel   flash-decoding: CTA = (kv head, 64-position split); K and V
//                        tiles arrive by bulk copy; scores thread = (head, position),
//                        P.V thread = (head, dim pair); (m, l, acc) per split
//   attn_oproj_kernel    every CTA merges the split partials in fixed order (bf16 o
//                        in smem), then warp-per-row GEMV over Wo (33.5 MB) + residual
#include <algorithm>

#include <cstdlib>

#include "common.cuh"

namespace daop {

constexpr int AT_WARPS = 16;    // GEMV CTAs

// profiling aid (daop_attn_timeline): global-timer span of each decode
// attention kernel's last launch -- [qkv, core, oproj][first CTA start, last
// CTA end] -- to see the gaps between the kernels of a decoder layer
// (per CTA, overwritten by every launch: the host takes min start / max end
// of the last launch of each kernel)
constexpr int AT_TL_CTAS = 256;
__device__ unsigned long long g_attn_tl[3][AT_TL_CTAS][2];
__device__ int g_attn_tl_on;
__device__ __forceinline__ void attn_tl(int k, int end) {
  const int b = blockIdx.x + blockIdx.y * gridDim.x;
  if (g_attn_tl_on && threadIdx.x == 0 && b < AT_TL_CTAS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_attn_tl[k][b][end] = t;
  }
}
constexpr int AT_HD = 128;      // head dim (Mixtral / Llama)
constexpr int AT_MAX_GROUP = 8; // q heads per kv head

// Bulk-streamed GEMV over this CTA's block of rows: warp AT_WARPS (lane 0)
// is the producer -- one cp.async.bulk per row into a ring of S = AT_WARPS
// row stages, issued from the first cycle of the kernel (the weights do not
// depend on x) -- and warps 0..AT_WARPS-1 consume rows round-robin (row i:
// stage and warp i % AT_WARPS, so each stage's phases are consumed in order
// by one warp): dot with x (smem) in a fixed lane-strided order + butterfly
// sum, then free the stage.
struct RowRing {
  uint8_t* ring;     // S x row_bytes
  uint64_t* full;    // S
  uint64_t* empty;   // S
  int S;
};

__device__ __forceinline__ void ring_init(RowRing& R) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < R.S; ++i) {
      mbar_init(&R.full[i], 1);
      mbar_init(&R.empty[i], 1);
    }
    fence_mbar_init();
  }
}

__device__ __forceinline__ void ring_produce(const RowRing& R, const uint16_t* W, int r0, int n,
                                             int K) {
  const uint32_t rb = static_cast<uint32_t>(K) * 2;
  for (int i = 0; i < n; ++i) {
    const int st = i % R.S;
    mbar_wait(&R.empty[st], ((i / R.S) & 1) ^ 1);
    mbar_arrive_expect_tx(&R.full[st], rb);
    bulk_g2s_plain(R.ring + static_cast<size_t>(st) * rb, W + static_cast<int64_t>(r0 + i) * K,
                   rb, &R.full[st]);
  }
}

template <class Epi>
__device__ __forceinline__ void ring_consume(const RowRing& R, int r0, int n, int K,
                                             const uint4* x_s, int warp, int lane, Epi epi) {
  const uint32_t rb = static_cast<uint32_t>(K) * 2;
  const int n16 = K / 8;
  for (int i = warp; i < n; i += AT_WARPS) {
    const int st = i % R.S;
    mbar_wait(&R.full[st], (i / R.S) & 1);
    const uint4* wr = reinterpret_cast<const uint4*>(R.ring + static_cast<size_t>(st) * rb);
    float acc = 0.f;
    for (int c = lane; c < n16; c += 32) acc = dot8(x_s[c], wr[c], acc);
    acc = warp_sum(acc);
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&R.empty[st]);
      epi(r0 + i, acc);
    }
  }
}

__global__ void __launch_bounds__((AT_WARPS + 1) * 32, 1)
    attn_qkv_kernel(const float* __restrict__ h, const uint16_t* __restrict__ gamma,
                    const uint16_t* __restrict__ wqkv, int d, int rows, int rows_per_cta,
                    int stages, float eps, uint16_t* __restrict__ xa_out,
                    float* __restrict__ qkv) {
  extern __shared__ __align__(128) uint8_t smem[];
  // the attention core (launched programmatically behind this grid) may start
  // now: its K / V loads do not depend on this kernel's output
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  attn_tl(0, 0);
  RowRing R;
  R.S = stages;
  R.ring = smem;
  uint16_t* xs = reinterpret_cast<uint16_t*>(smem + static_cast<size_t>(stages) * d * 2);
  double* red = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(xs) + d * 2);
  R.full = reinterpret_cast<uint64_t*>(red + 40);
  R.empty = R.full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * rows_per_cta;
  const int n = max(0, min(rows, r0 + rows_per_cta) - r0);
  ring_init(R);
  __syncthreads();
  if (warp == AT_WARPS) {  // producer warp: stream the rows while the others normalise
    if (lane == 0) ring_produce(R, wqkv, r0, n, d);
    return;
  }
  // RMSNorm by the consumer warps (named barrier: the producer is not waited
  // for).  Chunks of 8: h (2 x float4) and gamma (uint4) loaded once, up front;
  // <= 2 chunks per thread in registers (d <= 16 * AT_WARPS * 32), else reload.
  const int nt = AT_WARPS * 32, n8 = d / 8, tid = threadIdx.x;
  const float4* h4 = reinterpret_cast<const float4*>(h);
  const uint4* g4 = reinterpret_cast<const uint4*>(gamma);
  const bool regs = n8 <= 2 * nt;
  const int c0 = tid, c1 = tid + nt;
  // launched with programmatic stream serialization behind the previous
  // layer's MoE kernel: the producer warp above already streams Wqkv; h is
  // that kernel's output, read only after it completed (no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float4 ha = make_float4(0.f, 0.f, 0.f, 0.f), hb = ha, hc = ha, hd = ha;
  uint4 ga = make_uint4(0u, 0u, 0u, 0u), gb = ga;
  if (regs && c0 < n8) { ha = h4[2 * c0]; hb = h4[2 * c0 + 1]; ga = g4[c0]; }
  if (regs && c1 < n8) { hc = h4[2 * c1]; hd = h4[2 * c1 + 1]; gb = g4[c1]; }
  double ss = 0.0;  // fp64 squares: common.cuh rms_scale
  if (regs) {
    ss = sq_acc4(hd, sq_acc4(hc, sq_acc4(hb, sq_acc4(ha, ss))));
  } else {
    for (int i = tid; i < d; i += nt) ss = sq_acc(h[i], ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  asm volatile("bar.sync 1, %0;" ::"r"(nt));
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < AT_WARPS; ++w) t += red[w];
    red[32] = rms_scale(t, d, eps);
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nt));
  const float r = static_cast<float>(red[32]);
  auto norm8 = [&](int c, float4 u, float4 v, uint4 g) {
    const float hv[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
    uint32_t xw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float x0 = __fmul_rn(__fmul_rn(hv[2 * q], r), __uint_as_float(gw[q] << 16));
      const float x1 = __fmul_rn(__fmul_rn(hv[2 * q + 1], r), __uint_as_float(gw[q] & 0xffff0000u));
      xw[q] = static_cast<uint32_t>(f32_to_bf16_bits(x0)) |
              (static_cast<uint32_t>(f32_to_bf16_bits(x1)) << 16);
    }
    const uint4 x8 = make_uint4(xw[0], xw[1], xw[2], xw[3]);
    reinterpret_cast<uint4*>(xs)[c] = x8;
    if (xa_out && blockIdx.x == 0) reinterpret_cast<uint4*>(xa_out)[c] = x8;
  };
  if (regs) {
    if (c0 < n8) norm8(c0, ha, hb, ga);
    if (c1 < n8) norm8(c1, hc, hd, gb);
  } else {
    for (int c = tid; c < n8; c += nt) norm8(c, h4[2 * c], h4[2 * c + 1], g4[c]);
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nt));
  ring_consume(R, r0, n, d, reinterpret_cast<const uint4*>(xs), warp, lane,
               [&](int row, float v) { qkv[row] = v; });
  attn_tl(0, 1);
}

// RoPE of one head vector held as hd floats in smem (pairs (i, i + hd/2)).
// rope_inv / rope_angle / rope_apply are the pieces every kernel uses, in the
// same order with explicitly rounded operations, so a rotation computed from a
// shared cos / sin table is bit-identical to rope_pair's
__device__ __forceinline__ float rope_inv(int i, float theta) {
  return 1.0f / powf(theta, static_cast<float>(2 * i) / static_cast<float>(AT_HD));
}
__device__ __forceinline__ void rope_apply(float& a, float& b, float c, float s) {
  const float a2 = __fmaf_rn(a, c, -__fmul_rn(b, s));
  const float b2 = __fmaf_rn(b, c, __fmul_rn(a, s));
  a = a2;
  b = b2;
}
__device__ __forceinline__ void rope_pair(float& a, float& b, int i, int pos, float theta) {
  const float ang = __fmul_rn(static_cast<float>(pos), rope_inv(i, theta));
  float s, c;
  sincosf(ang, &s, &c);
  rope_apply(a, b, c, s);
}

struct AttnArgs {
  const float* qkv;       // raw projections: q (n_heads*hd) | k (n_kv*hd) | v (n_kv*hd)
  uint16_t* k_cache;      // (n_kv, max_seq, hd) bf16, this layer
  uint16_t* v_cache;
  int n_heads, n_kv, max_seq, pos, splits;
  float theta, scale;
  float* part;            // (n_kv, splits, group, 2 + hd): m, l, acc[hd]
  unsigned* counter;      // (n_kv) finished splits, self-resetting
  uint16_t* o;            // (n_heads * hd) bf16 attention output
};

constexpr int AT_SPLIT = 64;  // positions per CTA (one K tile + one V tile, 16 KB each)

// Shared-memory scratch of one attention split task
struct SplitSmem {
  __align__(128) uint16_t k_s[AT_SPLIT * AT_HD];
  __align__(128) uint16_t v_s[AT_SPLIT * AT_HD];
  float q_s[AT_MAX_GROUP][AT_HD];
  float p_s[AT_MAX_GROUP][AT_SPLIT];
  float ml_s[AT_MAX_GROUP][2];
  uint64_t bar;
  int last;
};

// One split task: kv head g, positions split * AT_SPLIT .. + AT_SPLIT - 1, on
// 256 threads (tid 0..255) that synchronise with `sync()` (__syncthreads in
// the standalone kernel, a named barrier in the fused one).  The split's K
// and V rows (contiguous in the cache) arrive by two bulk copies while the
// threads apply RoPE to the group's q heads; scores: thread = (head,
// position); P.V: thread = (head, 2 head dims).  The split's (m, l, acc) go to
// `part`; the task whose split holds `pos` first appends the new k (RoPE) and
// v.  The kv head's last split to finish merges all of them into o (fixed
// split order) and returns true.
template <class Sync>
__device__ __forceinline__ bool attn_split_task(const AttnArgs& a, int g, int split, int used,
                                                int tid, SplitSmem& S, Sync sync,
                                                unsigned* loaded = nullptr) {
  constexpr int NT = 256;
  const int lane = tid & 31;
  const int group = a.n_heads / a.n_kv;
  const int q_dim = a.n_heads * AT_HD, kv_dim = a.n_kv * AT_HD;
  const int p0 = split * AT_SPLIT;
  const int n = min(a.pos + 1, p0 + AT_SPLIT) - p0;  // positions of this split (>= 1)
  uint16_t* kc = a.k_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  uint16_t* vc = a.v_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  const bool owns_new = a.pos >= p0 && a.pos < p0 + AT_SPLIT;
  const int n_load = owns_new ? n - 1 : n;  // rows already in the cache
  uint16_t* k_s = S.k_s;
  uint16_t* v_s = S.v_s;
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    fence_mbar_init();
    if (n_load > 0) {
      mbar_arrive_expect_tx(&S.bar, 2 * n_load * AT_HD * 2);
      bulk_g2s_plain(k_s, kc + static_cast<int64_t>(p0) * AT_HD, n_load * AT_HD * 2, &S.bar);
      bulk_g2s_plain(v_s, vc + static_cast<int64_t>(p0) * AT_HD, n_load * AT_HD * 2, &S.bar);
    } else {
      mbar_arrive_expect_tx(&S.bar, 0);
    }
  }
  // launched programmatically behind the QKV GEMV: the cached K / V rows are
  // already on their way; q, k, v of this token are that kernel's output
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // q of the group's heads with RoPE
  for (int i = tid; i < group * (AT_HD / 2); i += NT) {
    const int hh = i / (AT_HD / 2), j = i - hh * (AT_HD / 2);
    float x0 = a.qkv[(g * group + hh) * AT_HD + j];
    float x1 = a.qkv[(g * group + hh) * AT_HD + j + AT_HD / 2];
    rope_pair(x0, x1, j, a.pos, a.theta);
    S.q_s[hh][j] = x0;
    S.q_s[hh][j + AT_HD / 2] = x1;
  }
  if (owns_new) {  // new k (RoPE) and v -> the cache and this task's tile
    const int r = a.pos - p0;
    for (int j = tid; j < AT_HD / 2; j += NT) {
      float k0 = a.qkv[q_dim + g * AT_HD + j];
      float k1 = a.qkv[q_dim + g * AT_HD + j + AT_HD / 2];
      rope_pair(k0, k1, j, a.pos, a.theta);
      const uint16_t b0 = f32_to_bf16_bits(k0), b1 = f32_to_bf16_bits(k1);
      kc[static_cast<int64_t>(a.pos) * AT_HD + j] = b0;
      kc[static_cast<int64_t>(a.pos) * AT_HD + j + AT_HD / 2] = b1;
      k_s[r * AT_HD + j] = b0;
      k_s[r * AT_HD + j + AT_HD / 2] = b1;
    }
    for (int j = tid; j < AT_HD; j += NT) {
      const uint16_t bv = f32_to_bf16_bits(a.qkv[q_dim + kv_dim + g * AT_HD + j]);
      vc[static_cast<int64_t>(a.pos) * AT_HD + j] = bv;
      v_s[r * AT_HD + j] = bv;
    }
  }
  sync();
  mbar_wait(&S.bar, 0);
  if (loaded && tid == 0) atomicAdd(loaded, 1u);  // fused kernel: this task's K / V landed
  // scores: thread = (head hh, position i); group * AT_SPLIT <= 512 -> two passes max
  for (int t = tid; t < group * AT_SPLIT; t += NT) {
    const int hh = t / AT_SPLIT, i = t - hh * AT_SPLIT;
    float sc = -INFINITY;
    if (i < n) {
      const uint4* kr = reinterpret_cast<const uint4*>(k_s + i * AT_HD);
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < AT_HD / 8; ++c) {
        const uint4 kv = kr[(c + i) & (AT_HD / 8 - 1)];  // rotated start: no bank conflicts
        const int cc = ((c + i) & (AT_HD / 8 - 1)) * 8;
        acc = fmaf(S.q_s[hh][cc + 0], bf16lo(kv.x), acc);
        acc = fmaf(S.q_s[hh][cc + 1], bf16hi(kv.x), acc);
        acc = fmaf(S.q_s[hh][cc + 2], bf16lo(kv.y), acc);
        acc = fmaf(S.q_s[hh][cc + 3], bf16hi(kv.y), acc);
        acc = fmaf(S.q_s[hh][cc + 4], bf16lo(kv.z), acc);
        acc = fmaf(S.q_s[hh][cc + 5], bf16hi(kv.z), acc);
        acc = fmaf(S.q_s[hh][cc + 6], bf16lo(kv.w), acc);
        acc = fmaf(S.q_s[hh][cc + 7], bf16hi(kv.w), acc);
      }
      sc = acc * a.scale;
    }
    S.p_s[hh][i] = sc;
  }
  sync();
  // per head: max and exp-sum over the split (one warp per head, fixed order)
  const int warp = tid >> 5;
  for (int hh = warp; hh < group; hh += NT / 32) {
    float mx = fmaxf(S.p_s[hh][lane], S.p_s[hh][lane + 32]);
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float e0 = lane < n ? expf(S.p_s[hh][lane] - mx) : 0.f;
    const float e1 = lane + 32 < n ? expf(S.p_s[hh][lane + 32] - mx) : 0.f;
    S.p_s[hh][lane] = e0;
    S.p_s[hh][lane + 32] = e1;
    const float se = warp_sum(e0 + e1);
    if (lane == 0) {
      S.ml_s[hh][0] = mx;
      S.ml_s[hh][1] = se;
    }
  }
  sync();
  // P.V: thread = (head hh, dims 2c, 2c + 1)
  for (int t = tid; t < group * (AT_HD / 2); t += NT) {
    const int hh = t / (AT_HD / 2), c = t - hh * (AT_HD / 2);
    float a0 = 0.f, a1 = 0.f;
    for (int i = 0; i < n; ++i) {
      const uint32_t vv = *reinterpret_cast<const uint32_t*>(v_s + i * AT_HD + 2 * c);
      a0 = fmaf(S.p_s[hh][i], bf16lo(vv), a0);
      a1 = fmaf(S.p_s[hh][i], bf16hi(vv), a1);
    }
    float* pr = a.part + ((static_cast<int64_t>(g) * a.splits + split) * group + hh) * (2 + AT_HD);
    pr[2 + 2 * c] = a0;
    pr[2 + 2 * c + 1] = a1;
    if (c == 0) {
      pr[0] = S.ml_s[hh][0];
      pr[1] = S.ml_s[hh][1];
    }
  }
  // the kv head's last split to finish merges all of them (fixed split order)
  __threadfence();
  sync();
  if (tid == 0) {
    S.last = atomicAdd(a.counter + g, 1u) == static_cast<unsigned>(used) - 1;
    if (S.last) a.counter[g] = 0;  // self-resetting for the next call
  }
  sync();
  const bool last = S.last;
  if (last) {
    __threadfence();
    for (int t = tid; t < group * (AT_HD / 2); t += NT) {
      const int hh = t / (AT_HD / 2), c = t - hh * (AT_HD / 2);
      const float* base = a.part + (static_cast<int64_t>(g) * a.splits * group + hh) * (2 + AT_HD);
      const int64_t stride = static_cast<int64_t>(group) * (2 + AT_HD);
      // the partials are read in batches of 8 splits with every load of a batch
      // issued before the first use (one L2 round trip per batch, not per split)
      constexpr int MB = 8;
      float m = -INFINITY;
      for (int s0 = 0; s0 < used; s0 += MB) {
        float mv[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) mv[j] = s0 + j < used ? __ldcg(base + (s0 + j) * stride) : -INFINITY;
#pragma unroll
        for (int j = 0; j < MB; ++j) m = fmaxf(m, mv[j]);
      }
      float l = 0.f, o0 = 0.f, o1 = 0.f;
      for (int s0 = 0; s0 < used; s0 += MB) {
        float mv[MB], lv[MB], a0[MB], a1[MB];
#pragma unroll
        for (int j = 0; j < MB; ++j) {
          const bool ok = s0 + j < used;
          const float* pr = base + (s0 + j) * stride;
          mv[j] = ok ? __ldcg(pr) : -INFINITY;
          lv[j] = ok ? __ldcg(pr + 1) : 0.f;
          a0[j] = ok ? __ldcg(pr + 2 + 2 * c) : 0.f;
          a1[j] = ok ? __ldcg(pr + 3 + 2 * c) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < MB; ++j) {  // fixed split order, as before
          if (s0 + j < used) {
            const float cf = expf(mv[j] - m);
            l = fmaf(lv[j], cf, l);
            o0 = fmaf(a0[j], cf, o0);
            o1 = fmaf(a1[j], cf, o1);
          }
        }
      }
      const int head = g * group + hh;
      a.o[head * AT_HD + 2 * c] = f32_to_bf16_bits(o0 / l);
      a.o[head * AT_HD + 2 * c + 1] = f32_to_bf16_bits(o1 / l);
    }
  }
  sync();  // the scratch (and S.bar) is reused by the next task
  if (tid == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&S.bar)) : "memory");
  return last;
}

// CTA = (kv head, split), 256 threads: attn_split_task
__global__ void __launch_bounds__(256, 1) attn_decode_kernel(AttnArgs a) {
  __shared__ SplitSmem S;
  // the O projection (launched programmatically behind this grid) may start
  // streaming Wo now; it waits for this grid before reading o
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  attn_tl(1, 0);
  attn_split_task(a, blockIdx.x, blockIdx.y, gridDim.y, threadIdx.x, S, [] { __syncthreads(); });
  attn_tl(1, 1);
}

// h' = h + o . Wo^T  (rows of Wo are output dims; o bf16 (q_dim) in smem)
__global__ void __launch_bounds__((AT_WARPS + 1) * 32, 1)
    attn_oproj_kernel(const float* __restrict__ h, const uint16_t* __restrict__ o,
                      const uint16_t* __restrict__ wo, int d, int q_dim, int rows_per_cta,
                      int stages, float* __restrict__ h_out) {
  extern __shared__ __align__(128) uint8_t smem[];
  RowRing R;
  R.S = stages;
  R.ring = smem;
  uint4* os = reinterpret_cast<uint4*>(smem + static_cast<size_t>(stages) * q_dim * 2);
  R.full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(os) + q_dim * 2);
  R.empty = R.full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * rows_per_cta;
  const int n = max(0, min(d, r0 + rows_per_cta) - r0);
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  attn_tl(2, 0);
  ring_init(R);
  __syncthreads();
  if (warp == AT_WARPS) {
    if (lane == 0) ring_produce(R, wo, r0, n, q_dim);
    return;
  }
  // launched programmatically behind the attention core: Wo is streaming;
  // o is that kernel's output (no-op for a plain launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = threadIdx.x; i < q_dim / 8; i += AT_WARPS * 32)
    os[i] = reinterpret_cast<const uint4*>(o)[i];
  asm volatile("bar.sync 1, %0;" ::"r"(AT_WARPS * 32));
  ring_consume(R, r0, n, q_dim, os, warp, lane,
               [&](int row, float v) { h_out[row] = h[row] + v; });
  attn_tl(2, 1);
}

// Attention core + O projection in ONE cooperative launch (one CTA per SM):
// every CTA's producer warp streams its Wo rows into the ring from the first
// cycle (the weights do not depend on o); CTAs < n_kv * used first run the
// attention split tasks on warps 0..7 (named barrier 2); the kv heads' last
// splits merge o and count the head; then every CTA waits for all n_kv heads,
// reads o and finishes the GEMV + residual as attn_oproj_kernel does.  The
// Wo stream overlaps the latency-bound attention core instead of starting
// after it.  sync[0] counts merged heads, sync[1] exits (the last CTA out
// resets both).
// attention core + O projection as two launches (default) or fused in one
// cooperative launch (DAOP_ATTN_FUSED=1 / 2, daop_set_attn_fused: measured
// slower -- 27.7-28.1 vs 25.3 us per attention layer at ctx 512, 36-37 vs 31
// at ctx 2000, also with the Wo stream held back until the split tasks' K / V
// landed (mode 2); DESIGN §6 tried table)
static int g_attn_fused = -1;
static int attn_fused_mode() {
  if (g_attn_fused < 0) {
    const char* v = getenv("DAOP_ATTN_FUSED");
    g_attn_fused = v ? atoi(v) : 0;
  }
  return g_attn_fused;
}

struct CoreOprojArgs {
  AttnArgs a;
  const float* h;
  const uint16_t* wo;
  int d, q_dim, rows_per_cta, stages, used;
  float* h_out;
  unsigned* sync;  // [0] merged heads, [1] exits, [2] split tasks whose K / V landed
  int delay;       // producer waits for the first wave's K / V (mode 2)
};

__global__ void __launch_bounds__((AT_WARPS + 1) * 32, 1) attn_core_oproj_kernel(CoreOprojArgs c) {
  extern __shared__ __align__(128) uint8_t smem[];
  RowRing R;
  R.S = c.stages;
  R.ring = smem;
  uint4* os = reinterpret_cast<uint4*>(smem + static_cast<size_t>(c.stages) * c.q_dim * 2);
  R.full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(os) + c.q_dim * 2);
  R.empty = R.full + c.stages;
  SplitSmem* S2 = reinterpret_cast<SplitSmem*>(
      reinterpret_cast<uint8_t*>(R.empty + c.stages) +
      ((128 - (reinterpret_cast<uintptr_t>(R.empty + c.stages) & 127)) & 127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * c.rows_per_cta;
  const int n = max(0, min(c.d, r0 + c.rows_per_cta) - r0);
  const int n_kv = c.a.n_kv, ntasks = n_kv * c.used;
  ring_init(R);
  __syncthreads();
  if (warp == AT_WARPS) {
    if (lane == 0) {
      // delayed stream (mode 2): start Wo once the first wave of split tasks
      // has its K / V in shared memory, so their latency-critical loads do
      // not queue behind 19 MB of weight traffic
      if (c.delay) {
        const unsigned wave = static_cast<unsigned>(min(ntasks, 2 * static_cast<int>(gridDim.x)));
        while (ld_acquire_gpu(c.sync + 2) < wave) __nanosleep(128);
      }
      ring_produce(R, c.wo, r0, n, c.q_dim);
    }
    return;
  }
  // two task slots per CTA: warps 0-7 (barrier 2) and 8-15 (barrier 3)
  const int slot = warp >> 3, tid = threadIdx.x & 255;
  for (int t = blockIdx.x + slot * gridDim.x; t < ntasks; t += 2 * gridDim.x) {
    const bool merged =
        slot == 0 ? attn_split_task(c.a, t / c.used, t % c.used, c.used, tid, S2[0],
                                    [] { asm volatile("bar.sync 2, 256;" ::: "memory"); }, c.sync + 2)
                  : attn_split_task(c.a, t / c.used, t % c.used, c.used, tid, S2[1],
                                    [] { asm volatile("bar.sync 3, 256;" ::: "memory"); }, c.sync + 2);
    if (merged && tid == 0) {  // o rows of this kv head are written
      __threadfence();
      atomicAdd(c.sync, 1u);
    }
  }
  if (threadIdx.x == 0)
    while (ld_acquire_gpu(c.sync) < static_cast<unsigned>(n_kv)) __nanosleep(64);
  asm volatile("bar.sync 1, %0;" ::"r"(AT_WARPS * 32));
  for (int i = threadIdx.x; i < c.q_dim / 8; i += AT_WARPS * 32)
    os[i] = __ldcg(reinterpret_cast<const uint4*>(c.a.o) + i);
  asm volatile("bar.sync 1, %0;" ::"r"(AT_WARPS * 32));
  ring_consume(R, r0, n, c.q_dim, os, warp, lane,
               [&](int row, float v) { c.h_out[row] = c.h[row] + v; });
  if (threadIdx.x == 0 && atomicAdd(c.sync + 1, 1u) == gridDim.x - 1) {
    c.sync[0] = 0;  // every CTA is past its waits: reset for the next call
    c.sync[2] = 0;
    __threadfence();
    c.sync[1] = 0;
  }
}

// ---------------------------------------------------------------------------
// Prefill: T prompt tokens of one layer at positions pos0 .. pos0 + T - 1.
// The projections are plain GEMMs over the T rows (the caller's cuBLAS calls:
// xa . Wqkv^T and o . Wo^T with fp32 output); these kernels do the rest.

// xa[t] = bf16(rmsnorm(h[t]) * gamma): one CTA per token
__global__ void __launch_bounds__(256) attn_norm_rows_kernel(const float* __restrict__ h,
                                                             const uint16_t* __restrict__ gamma,
                                                             int d, float eps,
                                                             uint16_t* __restrict__ xa) {
  pdl_prologue();  // (launched with launch_pdl)
  __shared__ double red[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n8 = d / 8;
  const float4* h4 = reinterpret_cast<const float4*>(h + static_cast<int64_t>(blockIdx.x) * d);
  const uint4* g4 = reinterpret_cast<const uint4*>(gamma);
  double ss = 0.0;  // fp64 squares: common.cuh rms_scale
  for (int c = tid; c < n8; c += blockDim.x) ss = sq_acc4(h4[2 * c + 1], sq_acc4(h4[2 * c], ss));
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float r = rms_scale(tot, d, eps);
  uint4* x4 = reinterpret_cast<uint4*>(xa + static_cast<int64_t>(blockIdx.x) * d);
  for (int c = tid; c < n8; c += blockDim.x) {
    const float4 u = h4[2 * c], v = h4[2 * c + 1];
    const uint4 g = g4[c];
    const float hv[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
    uint32_t xw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float x0 = __fmul_rn(__fmul_rn(hv[2 * q], r), __uint_as_float(gw[q] << 16));
      const float x1 = __fmul_rn(__fmul_rn(hv[2 * q + 1], r), __uint_as_float(gw[q] & 0xffff0000u));
      xw[q] = static_cast<uint32_t>(f32_to_bf16_bits(x0)) |
              (static_cast<uint32_t>(f32_to_bf16_bits(x1)) << 16);
    }
    x4[c] = make_uint4(xw[0], xw[1], xw[2], xw[3]);
  }
}

struct PrefillArgs {
  const float* qkv;   // (T, q_dim + 2 kv_dim) fp32, unrotated
  uint16_t* k_cache;  // (n_kv, max_seq, hd) bf16, this layer
  uint16_t* v_cache;
  int n_heads, n_kv, max_seq, pos0;
  float theta, scale;
  uint16_t* o;        // (T, n_heads * hd) bf16
};

// k (RoPE) and v of every prompt token -> the cache (before any attention
// reads it): CTA = token
__global__ void __launch_bounds__(128) attn_prefill_append_kernel(PrefillArgs a) {
  pdl_prologue();  // (launched with launch_pdl)
  const int t = blockIdx.x, p = a.pos0 + t;
  const int q_dim = a.n_heads * AT_HD, kv_dim = a.n_kv * AT_HD;
  const float* row = a.qkv + static_cast<int64_t>(t) * (q_dim + 2 * kv_dim);
  for (int i = threadIdx.x; i < a.n_kv * (AT_HD / 2); i += blockDim.x) {
    const int g = i / (AT_HD / 2), j = i - g * (AT_HD / 2);
    float k0 = row[q_dim + g * AT_HD + j], k1 = row[q_dim + g * AT_HD + j + AT_HD / 2];
    rope_pair(k0, k1, j, p, a.theta);
    uint16_t* kc = a.k_cache + (static_cast<int64_t>(g) * a.max_seq + p) * AT_HD;
    kc[j] = f32_to_bf16_bits(k0);
    kc[j + AT_HD / 2] = f32_to_bf16_bits(k1);
  }
  for (int i = threadIdx.x; i < kv_dim; i += blockDim.x) {
    const int g = i / AT_HD, j = i - g * AT_HD;
    a.v_cache[(static_cast<int64_t>(g) * a.max_seq + p) * AT_HD + j] =
        f32_to_bf16_bits(row[q_dim + kv_dim + i]);
  }
}

// causal attention of query token t (position pos0 + t) over positions
// 0 .. pos0 + t: CTA = (kv head g, token t); 64-position K / V tiles by bulk
// copy; per tile the same scores / exp / P.V as attn_decode_kernel's split,
// folded into running (m, l, acc) with the usual rescaling
__global__ void __launch_bounds__(256, 2) attn_prefill_kernel(PrefillArgs a) {
  __shared__ __align__(128) uint16_t k_s[AT_SPLIT * AT_HD];
  __shared__ __align__(128) uint16_t v_s[AT_SPLIT * AT_HD];
  __shared__ float q_s[AT_MAX_GROUP][AT_HD];
  __shared__ float p_s[AT_MAX_GROUP][AT_SPLIT];
  __shared__ float ml_s[AT_MAX_GROUP][2];
  __shared__ uint64_t bar;
  const int g = blockIdx.x, t = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const int p = a.pos0 + t;
  const int group = a.n_heads / a.n_kv;
  const int q_dim = a.n_heads * AT_HD, kv_dim = a.n_kv * AT_HD;
  const float* row = a.qkv + static_cast<int64_t>(t) * (q_dim + 2 * kv_dim);
  const uint16_t* kc = a.k_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  const uint16_t* vc = a.v_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < group * (AT_HD / 2); i += blockDim.x) {
    const int hh = i / (AT_HD / 2), j = i - hh * (AT_HD / 2);
    float x0 = row[(g * group + hh) * AT_HD + j];
    float x1 = row[(g * group + hh) * AT_HD + j + AT_HD / 2];
    rope_pair(x0, x1, j, p, a.theta);
    q_s[hh][j] = x0;
    q_s[hh][j + AT_HD / 2] = x1;
  }
  // running state of this thread's (head, dim pair) items (<= 2: group <= 8)
  constexpr int MAXI = AT_MAX_GROUP * (AT_HD / 2) / 256;
  float rm[MAXI], rl[MAXI], o0[MAXI], o1[MAXI];
#pragma unroll
  for (int q = 0; q < MAXI; ++q) rm[q] = -INFINITY, rl[q] = o0[q] = o1[q] = 0.f;
  const int tiles = p / AT_SPLIT + 1;
  for (int s = 0; s < tiles; ++s) {
    const int p0 = s * AT_SPLIT;
    const int n = min(p + 1, p0 + AT_SPLIT) - p0;
    __syncthreads();  // the previous tile is fully consumed (and q_s / bar are ready)
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar, 2 * n * AT_HD * 2);
      bulk_g2s_plain(k_s, kc + static_cast<int64_t>(p0) * AT_HD, n * AT_HD * 2, &bar);
      bulk_g2s_plain(v_s, vc + static_cast<int64_t>(p0) * AT_HD, n * AT_HD * 2, &bar);
    }
    mbar_wait(&bar, s & 1);
    for (int u = tid; u < group * AT_SPLIT; u += blockDim.x) {
      const int hh = u / AT_SPLIT, i = u - hh * AT_SPLIT;
      float sc = -INFINITY;
      if (i < n) {
        const uint4* kr = reinterpret_cast<const uint4*>(k_s + i * AT_HD);
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < AT_HD / 8; ++c) {
          const uint4 kv = kr[(c + i) & (AT_HD / 8 - 1)];
          const int cc = ((c + i) & (AT_HD / 8 - 1)) * 8;
          acc = fmaf(q_s[hh][cc + 0], bf16lo(kv.x), acc);
          acc = fmaf(q_s[hh][cc + 1], bf16hi(kv.x), acc);
          acc = fmaf(q_s[hh][cc + 2], bf16lo(kv.y), acc);
          acc = fmaf(q_s[hh][cc + 3], bf16hi(kv.y), acc);
          acc = fmaf(q_s[hh][cc + 4], bf16lo(kv.z), acc);
          acc = fmaf(q_s[hh][cc + 5], bf16hi(kv.z), acc);
          acc = fmaf(q_s[hh][cc + 6], bf16lo(kv.w), acc);
          acc = fmaf(q_s[hh][cc + 7], bf16hi(kv.w), acc);
        }
        sc = acc * a.scale;
      }
      p_s[hh][i] = sc;
    }
    __syncthreads();
    const int warp = tid >> 5;
    for (int hh = warp; hh < group; hh += blockDim.x / 32) {
      float mx = fmaxf(p_s[hh][lane], p_s[hh][lane + 32]);
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float e0 = lane < n ? expf(p_s[hh][lane] - mx) : 0.f;
      const float e1 = lane + 32 < n ? expf(p_s[hh][lane + 32] - mx) : 0.f;
      p_s[hh][lane] = e0;
      p_s[hh][lane + 32] = e1;
      const float se = warp_sum(e0 + e1);
      if (lane == 0) {
        ml_s[hh][0] = mx;
        ml_s[hh][1] = se;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < MAXI; ++q) {
      const int u = tid + q * blockDim.x;
      if (u >= group * (AT_HD / 2)) break;
      const int hh = u / (AT_HD / 2), c = u - hh * (AT_HD / 2);
      float a0 = 0.f, a1 = 0.f;
      for (int i = 0; i < n; ++i) {
        const uint32_t vv = *reinterpret_cast<const uint32_t*>(v_s + i * AT_HD + 2 * c);
        a0 = fmaf(p_s[hh][i], bf16lo(vv), a0);
        a1 = fmaf(p_s[hh][i], bf16hi(vv), a1);
      }
      const float ms = ml_s[hh][0], mn = fmaxf(rm[q], ms);
      const float co = expf(rm[q] - mn), cs = expf(ms - mn);  // rm = -inf -> co = 0
      rl[q] = fmaf(rl[q], co, ml_s[hh][1] * cs);
      o0[q] = fmaf(o0[q], co, a0 * cs);
      o1[q] = fmaf(o1[q], co, a1 * cs);
      rm[q] = mn;
    }
  }
#pragma unroll
  for (int q = 0; q < MAXI; ++q) {
    const int u = tid + q * blockDim.x;
    if (u >= group * (AT_HD / 2)) break;
    const int hh = u / (AT_HD / 2), c = u - hh * (AT_HD / 2);
    uint16_t* orow = a.o + static_cast<int64_t>(t) * q_dim + (g * group + hh) * AT_HD;
    orow[2 * c] = f32_to_bf16_bits(o0[q] / rl[q]);
    orow[2 * c + 1] = f32_to_bf16_bits(o1[q] / rl[q]);
  }
}

// ---------------------------------------------------------------------------
// Causal prompt attention on the tensor cores (FlashAttention-2 style).
// CTA = (kv head g, 16 query tokens); warp w = query head g * group + w, so
// the GQA group's heads share every K / V tile the CTA stages.  Per warp:
//   Q (16 x 128) = bf16(RoPE(q)) held as m16n8k16 A fragments (32 regs);
//   per 64-position tile: S = Q K^T (ldmatrix B fragments from the padded
//   K tile), causal mask, online softmax in fp32 (running max / sum per row,
//   the accumulator rescaled), P = bf16(exp(S - m)) reused in registers as
//   the A operand of O += P V (V fragments by ldmatrix.trans);
//   o = bf16(O / l).
// K / V tiles (64 x 128 bf16, rows padded to 136 elements: conflict-free
// ldmatrix) are double-buffered with cp.async.  Numerics vs the oracle
// (oracle/numerics.attention_decode): q and P are rounded to bf16 for the
// MMAs (fp32 accumulation); within the hidden-state tolerance (tests).
constexpr int FA_TOK = 16;            // query tokens per CTA (MMA M)
constexpr int FA_KV = 64;             // positions per K / V tile
constexpr int FA_LD = AT_HD + 8;      // padded smem row (bf16 elements)
constexpr int FA_TILE = FA_KV * FA_LD;  // elements of one K (or V) tile

__device__ __forceinline__ void mma_bf16_16816_acc(float (&d)[4], uint32_t a0, uint32_t a1,
                                                   uint32_t a2, uint32_t a3, uint32_t b0,
                                                   uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  // invalid rows are zero-filled (src-size 0): masked positions never read garbage
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)),
               "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  return static_cast<uint32_t>(f32_to_bf16_bits(lo)) |
         (static_cast<uint32_t>(f32_to_bf16_bits(hi)) << 16);
}

// KV split (FA_HALVES = 2 when 2 x group warps fit 256 threads): the group's
// warps run twice, half h over the K / V tiles [h * n0, ...) of the CTA's
// causal range with its own two-stage buffers and named barrier; half 1's
// (m, l, O) are merged into half 0's at the end (flash-decoding style), which
// halves the serial tile loop of the late token tiles -- the kernel's
// critical path (the last 16 tokens see all 4 tiles of a 256-token prompt).
constexpr int FA_HALVES_MAX = 2;
__global__ void __launch_bounds__(256) attn_prefill_mma_kernel(PrefillArgs a, int T) {
  pdl_prologue();  // (launched with launch_pdl)
  extern __shared__ __align__(128) uint16_t fa_smem[];  // [2 stages][K | V] tiles
  const int g = blockIdx.x, t0 = blockIdx.y * FA_TOK;
  const int group = a.n_heads / a.n_kv;
  const int halves = static_cast<int>(blockDim.x) / (group * 32);  // 1 or 2
  const int warp_all = threadIdx.x >> 5, lane = threadIdx.x & 31, nthr_all = blockDim.x;
  const int half = warp_all / group, warp = warp_all - half * group, nthr = group * 32;
  const int htid = threadIdx.x - half * nthr;  // thread index within the half
  const int gr = lane >> 2, c4 = lane & 3;  // fragment row / column pair
  const int q_dim = a.n_heads * AT_HD, kv_dim = a.n_kv * AT_HD, ld = q_dim + 2 * kv_dim;
  const int hh = g * group + warp;  // this warp's query head
  const uint16_t* kc = a.k_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  const uint16_t* vc = a.v_cache + static_cast<int64_t>(g) * a.max_seq * AT_HD;
  const int t_last = min(T, t0 + FA_TOK) - 1;
  const int n_pos = a.pos0 + t_last + 1;  // positions any row of this CTA attends to
  const int n_all = (n_pos + FA_KV - 1) / FA_KV;
  const int n_first = halves == 2 ? (n_all + 1) / 2 : n_all;  // half 0: [0, n_first)
  const int s_begin = half == 0 ? 0 : n_first, s_end = half == 0 ? n_first : n_all;
  uint16_t* const hsm = fa_smem + static_cast<size_t>(half) * 4 * FA_TILE;  // this half's stages
  auto hsync = [&] { asm volatile("bar.sync %0, %1;" ::"r"(1 + half), "r"(nthr) : "memory"); };

  auto load_tile = [&](int s) {  // positions [s * 64, s * 64 + 64) -> stage s & 1 of this half
    uint16_t* ks = hsm + (s & 1) * 2 * FA_TILE;
    uint16_t* vs = ks + FA_TILE;
    const int p0 = s * FA_KV;
    for (int i = htid; i < FA_KV * (AT_HD / 8); i += nthr) {
      const int r = i >> 4, c = (i & 15) * 8;
      const bool ok = p0 + r < n_pos;
      const int64_t src = static_cast<int64_t>(ok ? p0 + r : 0) * AT_HD + c;
      cp_async16(ks + r * FA_LD + c, kc + src, ok);
      cp_async16(vs + r * FA_LD + c, vc + src, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // the CTA's 16 token rows x the group's query heads staged in shared memory
  // by coalesced 16-byte copies (each thread used to issue 64 scalar loads of
  // its fragment elements: the kernel's top stall, lg_throttle / long
  // scoreboard); row stride padded so the fragment reads spread over banks
  const int q_ld = group * AT_HD + 8;
  float* const q_s = reinterpret_cast<float*>(fa_smem + static_cast<size_t>(halves) * 4 * FA_TILE);
  for (int i = threadIdx.x; i < FA_TOK * group * (AT_HD / 4); i += nthr_all) {
    const int r = i / (group * (AT_HD / 4)), c = (i - r * (group * (AT_HD / 4))) * 4;
    const int t = min(t0 + r, T - 1);
    cp_async16(q_s + r * q_ld + c, a.qkv + static_cast<int64_t>(t) * ld + g * group * AT_HD + c, true);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  if (s_begin < s_end) load_tile(s_begin);

  // the CTA's 16 tokens x 64 RoPE frequencies: cos / sin computed once and
  // shared by the group's warps (each warp used to evaluate powf + sincosf for
  // all 32 of its (row, dim) pairs -- 4x redundant, the kernel's longest phase)
  __shared__ float inv_s[AT_HD / 2];
  __shared__ float2 rope_cs[FA_TOK][AT_HD / 2];
  if (threadIdx.x < AT_HD / 2) inv_s[threadIdx.x] = rope_inv(threadIdx.x, a.theta);
  __syncthreads();
  for (int i = threadIdx.x; i < FA_TOK * (AT_HD / 2); i += nthr_all) {
    const int r = i / (AT_HD / 2), j = i - r * (AT_HD / 2);
    const int t = min(t0 + r, T - 1);
    float sn, cs;
    sincosf(__fmul_rn(static_cast<float>(a.pos0 + t), inv_s[j]), &sn, &cs);
    rope_cs[r][j] = make_float2(cs, sn);
  }
  if (s_begin < s_end) asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // Q, not tile s_begin
  else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // Q fragments: rows gr / gr + 8 = tokens t0 + gr / t0 + gr + 8; k-step ks
  // covers dims 16 ks .. 16 ks + 15; RoPE pairs (j, j + 64) = (ks, ks + 4)
  uint32_t qf[8][4];
  {
    float qv[2][8][4];  // [row half][ks][0..3] = dims 16ks + 2c4 + {0, 1, 8, 9}
#pragma unroll
    for (int rh = 0; rh < 2; ++rh) {
      const float* q = q_s + (gr + 8 * rh) * q_ld + warp * AT_HD;  // row clamped at staging
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = 16 * ks + 2 * c4 + (e & 1) + 8 * (e >> 1);  // j < 64
          float x0 = q[j], x1 = q[j + AT_HD / 2];
          const float2 cs = rope_cs[min(gr + 8 * rh, T - 1 - t0)][j];  // (row clamped like t)
          rope_apply(x0, x1, cs.x, cs.y);
          qv[rh][ks][e] = x0;
          qv[rh][ks + 4][e] = x1;
        }
    }
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qf[ks][0] = pack_bf16x2(qv[0][ks][0], qv[0][ks][1]);
      qf[ks][1] = pack_bf16x2(qv[1][ks][0], qv[1][ks][1]);
      qf[ks][2] = pack_bf16x2(qv[0][ks][2], qv[0][ks][3]);
      qf[ks][3] = pack_bf16x2(qv[1][ks][2], qv[1][ks][3]);
    }
  }
  const int lim0 = a.pos0 + min(t0 + gr, T - 1);      // last position row gr may see
  const int lim1 = a.pos0 + min(t0 + gr + 8, T - 1);  // ... row gr + 8
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int s = s_begin; s < s_end; ++s) {
    if (s + 1 < s_end) {
      load_tile(s + 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    hsync();
    const uint16_t* ks_ = hsm + (s & 1) * 2 * FA_TILE;
    const uint16_t* vs_ = ks_ + FA_TILE;
    const int p0 = s * FA_KV;
    // ---- S = Q K^T (16 x 64)
    float sc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int ks = 0; ks < 8; ks += 2) {
        const int mi = lane >> 3;
        const uint32_t addr = smem_u32(ks_ + (8 * j + (lane & 7)) * FA_LD + 16 * ks + 8 * mi);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(addr, b0, b1, b2, b3);
        mma_bf16_16816_acc(sc[j], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b0, b1);
        mma_bf16_16816_acc(sc[j], qf[ks + 1][0], qf[ks + 1][1], qf[ks + 1][2], qf[ks + 1][3], b2,
                           b3);
      }
    }
    // ---- scale, causal mask, online softmax (rows gr, gr + 8; a quad owns a row)
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int pos = p0 + 8 * j + 2 * c4 + e;
        sc[j][e] = pos <= lim0 ? sc[j][e] * a.scale : -INFINITY;
        sc[j][2 + e] = pos <= lim1 ? sc[j][2 + e] * a.scale : -INFINITY;
        mx0 = fmaxf(mx0, sc[j][e]);
        mx1 = fmaxf(mx1, sc[j][2 + e]);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    // half 0 sees position 0 in its first tile, so its mx is finite from
    // tile 0; half 1's first tile can be fully masked for some rows (mx stays
    // -inf: guard the rescale, e^(-inf - -inf))
    const float al0 = mx0 == -INFINITY ? 1.f : expf(m0 - mx0);
    const float al1 = mx1 == -INFINITY ? 1.f : expf(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        sc[j][e] = m0 == -INFINITY ? 0.f : expf(sc[j][e] - m0);
        sc[j][2 + e] = m1 == -INFINITY ? 0.f : expf(sc[j][2 + e] - m1);
        rs0 += sc[j][e];
        rs1 += sc[j][2 + e];
      }
    rs0 += __shfl_xor_sync(0xffffffffu, rs0, 1);
    rs0 += __shfl_xor_sync(0xffffffffu, rs0, 2);
    rs1 += __shfl_xor_sync(0xffffffffu, rs1, 1);
    rs1 += __shfl_xor_sync(0xffffffffu, rs1, 2);
    l0 = l0 * al0 + rs0;
    l1 = l1 * al1 + rs1;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= al0;
      o[i][1] *= al0;
      o[i][2] *= al1;
      o[i][3] *= al1;
    }
    // ---- O += P V: k-step kk = positions 16 kk .. 16 kk + 15 = S tiles 2kk, 2kk+1
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t pa0 = pack_bf16x2(sc[2 * kk][0], sc[2 * kk][1]);
      const uint32_t pa1 = pack_bf16x2(sc[2 * kk][2], sc[2 * kk][3]);
      const uint32_t pa2 = pack_bf16x2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
      const uint32_t pa3 = pack_bf16x2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
      for (int dn = 0; dn < 16; dn += 2) {
        const int mi = lane >> 3;
        const uint32_t addr =
            smem_u32(vs_ + (16 * kk + 8 * (mi & 1) + (lane & 7)) * FA_LD + 8 * (dn + (mi >> 1)));
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(addr, b0, b1, b2, b3);
        mma_bf16_16816_acc(o[dn], pa0, pa1, pa2, pa3, b0, b1);
        mma_bf16_16816_acc(o[dn + 1], pa0, pa1, pa2, pa3, b2, b3);
      }
    }
    hsync();  // this stage is refilled two iterations from now
  }
  if (halves == 2) {  // half 1's (m, l, O) -> shared memory; half 0 merges
    float* xch = reinterpret_cast<float*>(fa_smem + 4 * FA_TILE);  // half 1's stages (idle now)
    float* mine = xch + static_cast<size_t>(warp * 32 + lane) * 68;
    __syncthreads();
    if (half == 1) {
      mine[0] = m0;
      mine[1] = m1;
      mine[2] = l0;
      mine[3] = l1;
#pragma unroll
      for (int i = 0; i < 16; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) mine[4 + 4 * i + c] = o[i][c];
    }
    __syncthreads();
    if (half == 1) return;
    const float mb0 = mine[0], mb1 = mine[1], lb0 = mine[2], lb1 = mine[3];
    const float mm0 = fmaxf(m0, mb0), mm1 = fmaxf(m1, mb1);
    const float fa0 = expf(m0 - mm0), fa1 = expf(m1 - mm1);
    const float fb0 = mb0 == -INFINITY ? 0.f : expf(mb0 - mm0);
    const float fb1 = mb1 == -INFINITY ? 0.f : expf(mb1 - mm1);
    l0 = l0 * fa0 + lb0 * fb0;
    l1 = l1 * fa1 + lb1 * fb1;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] = o[i][0] * fa0 + mine[4 + 4 * i + 0] * fb0;
      o[i][1] = o[i][1] * fa0 + mine[4 + 4 * i + 1] * fb0;
      o[i][2] = o[i][2] * fa1 + mine[4 + 4 * i + 2] * fb1;
      o[i][3] = o[i][3] * fa1 + mine[4 + 4 * i + 3] * fb1;
    }
  }
  // ---- o = bf16(O / l) -> (T, q_dim) at this head's 128 columns
  const float inv0 = 1.0f / l0, inv1 = 1.0f / l1;
  const int ta = t0 + gr, tb = t0 + gr + 8;
#pragma unroll
  for (int dn = 0; dn < 16; ++dn) {
    const int col = hh * AT_HD + 8 * dn + 2 * c4;
    if (ta < T)
      *reinterpret_cast<uint32_t*>(a.o + static_cast<int64_t>(ta) * q_dim + col) =
          pack_bf16x2(o[dn][0] * inv0, o[dn][1] * inv0);
    if (tb < T)
      *reinterpret_cast<uint32_t*>(a.o + static_cast<int64_t>(tb) * q_dim + col) =
          pack_bf16x2(o[dn][2] * inv1, o[dn][3] * inv1);
  }
}

// L2 prefetch of up to two byte ranges (the next layer's attention weights,
// issued just before this layer's MoE decode kernel): the MoE kernel streams
// its experts with L2::evict_first, so the prefetched lines survive it and
// the next QKV / O-proj GEMVs read L2 instead of ramping up on HBM
constexpr int64_t PF_CHUNK = 32 * 1024;
__global__ void l2_prefetch_kernel(const uint8_t* __restrict__ p0, int64_t n0,
                                   const uint8_t* __restrict__ p1, int64_t n1) {
  const int64_t c0 = (n0 + PF_CHUNK - 1) / PF_CHUNK, c1 = (n1 + PF_CHUNK - 1) / PF_CHUNK;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < c0 + c1;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint8_t* p = c < c0 ? p0 + c * PF_CHUNK : p1 + (c - c0) * PF_CHUNK;
    const int64_t rem = c < c0 ? n0 - c * PF_CHUNK : n1 - (c - c0) * PF_CHUNK;
    const uint32_t bytes = static_cast<uint32_t>(rem < PF_CHUNK ? rem : PF_CHUNK);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)),
                 "r"(bytes)
                 : "memory");
  }
}

}  // namespace daop

using namespace daop;

extern "C" int daop_attn_norm_rows(const float* d_h, int64_t T, const uint16_t* d_gamma, int32_t d,
                                   float eps, uint16_t* d_xa, daop_stream_t stream) {
  if (T < 0 || d <= 0 || d % 8 != 0) {
    set_error("attn_norm_rows: unsupported shape (T=%lld, d=%d)", (long long)T, d);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (T == 0) return DAOP_OK;
  DAOP_CUDA(launch_pdl(attn_norm_rows_kernel, dim3(static_cast<unsigned>(T)), dim3(256), 0, as_stream(stream), d_h, d_gamma, d,
                                                                                 eps, d_xa));
  DAOP_CHECK_LAUNCH("attn_norm_rows");
  return DAOP_OK;
}

extern "C" int daop_attn_prefill(const float* d_qkv, int64_t T, int32_t pos0, uint16_t* d_k_cache,
                                 uint16_t* d_v_cache, int32_t n_heads, int32_t n_kv,
                                 int32_t max_seq, float theta, uint16_t* d_o,
                                 daop_stream_t stream) {
  if (n_kv < 1 || n_heads % n_kv != 0 || n_heads / n_kv > AT_MAX_GROUP || T < 0 || pos0 < 0 ||
      pos0 + T > max_seq || T > 65535) {
    set_error("attn_prefill: unsupported (heads=%d kv=%d pos0=%d T=%lld max_seq=%d)", n_heads,
              n_kv, pos0, (long long)T, max_seq);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (T == 0) return DAOP_OK;
  cudaStream_t st = as_stream(stream);
  PrefillArgs a{d_qkv, d_k_cache, d_v_cache, n_heads, n_kv, max_seq, pos0,
                theta, 1.0f / sqrtf(static_cast<float>(AT_HD)), d_o};
  DAOP_CUDA(launch_pdl(attn_prefill_append_kernel, dim3(static_cast<unsigned>(T)), dim3(128), 0, st, a));
  DAOP_CHECK_LAUNCH("attn_prefill_append");
  // KV split over two warp groups when 2 x group warps fit the 256-thread CTA
  // and the prompt spans more than one K / V tile (DAOP_ATTN_KV_SPLIT=0: off)
  static const bool kv_split = [] {
    const char* v = getenv("DAOP_ATTN_KV_SPLIT");
    return !(v && v[0] == '0');
  }();
  const int group = n_heads / n_kv;
  const int halves = kv_split && group * 64 <= 256 && pos0 + T > FA_KV ? FA_HALVES_MAX : 1;
  const size_t smem = static_cast<size_t>(halves) * 2 * 2 * FA_TILE * 2 +  // per half: 2 stages x (K, V)
                      static_cast<size_t>(FA_TOK) * (group * AT_HD + 8) * 4;    // + staged fp32 Q rows
  DAOP_CUDA(cudaFuncSetAttribute(attn_prefill_mma_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const unsigned tok_tiles = static_cast<unsigned>((T + FA_TOK - 1) / FA_TOK);
  DAOP_CUDA(launch_pdl(attn_prefill_mma_kernel, dim3(dim3(n_kv, tok_tiles)),
                       dim3(halves * group * 32), smem, st, a, static_cast<int>(T)));
  DAOP_CHECK_LAUNCH("attn_prefill");
  return DAOP_OK;
}

extern "C" int daop_attn_workspace(int32_t n_heads, int32_t n_kv, int32_t max_seq,
                                   int64_t* h_bytes) {
  // qkv fp32 | partials (n_kv x splits(<=64) x group x (2 + hd)) | o bf16
  const int64_t q_dim = static_cast<int64_t>(n_heads) * AT_HD;
  const int64_t kv_dim = static_cast<int64_t>(n_kv) * AT_HD;
  const int64_t part = static_cast<int64_t>(n_kv) * 64 * (n_heads / n_kv) * (2 + AT_HD) * 4;
  *h_bytes = (q_dim + 2 * kv_dim) * 4 + part + q_dim * 2 + 4 * n_kv + 128 + 12 + 256;  // + fused-kernel sync line
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
  unsigned* counter = reinterpret_cast<unsigned*>(o + q_dim);
  {
    const int rows = q_dim + 2 * kv_dim;
    const int rpc = (rows + sms - 1) / sms;
    // one stage per consumer warp: row i lives in stage i % AT_WARPS and is
    // consumed by warp i % AT_WARPS, so no warp can wait on a stage a whole
    // ring cycle ahead of its data (a shared ring would let it)
    const int stages = AT_WARPS;
    const size_t smem = static_cast<size_t>(stages) * d * 2 + static_cast<size_t>(d) * 2 + 40 * 8 +
                        2 * stages * 8;
    DAOP_CUDA(cudaFuncSetAttribute(attn_qkv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    static const int pdl = [] {
      const char* v = getenv("DAOP_ATTN_PDL");
      return v ? atoi(v) : 1;
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3((AT_WARPS + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    DAOP_CUDA(cudaLaunchKernelEx(&cfg, attn_qkv_kernel, d_h, d_gamma, d_wqkv, d, rows, rpc, stages,
                                 eps, d_xa_out, qkv));
    DAOP_CHECK_LAUNCH("attn_qkv");
  }
  // position splits of AT_SPLIT positions (<= 64 splits: max_seq <= 4096)
  const int ctx = pos + 1;
  const int used = (ctx + AT_SPLIT - 1) / AT_SPLIT;
  const int splits = 64;
  if (used > splits) {
    set_error("attention: context %d exceeds %d positions", ctx, splits * AT_SPLIT);
    return DAOP_ERR_UNSUPPORTED;
  }
  AttnArgs a{qkv, d_k_cache, d_v_cache, n_heads, n_kv, max_seq, pos, splits,
             theta, 1.0f / sqrtf(static_cast<float>(AT_HD)), part, counter, o};
  if (attn_fused_mode()) {  // attention core + O projection in one cooperative launch
    const int rpc = (d + sms - 1) / sms;
    const int stages = AT_WARPS;
    const size_t smem = static_cast<size_t>(stages) * q_dim * 2 + static_cast<size_t>(q_dim) * 2 +
                        2 * stages * 8 + 128 + 2 * sizeof(SplitSmem);
    DAOP_CUDA(cudaFuncSetAttribute(attn_core_oproj_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    // (the fused kernel's polled words on their own 128-byte line, away from
    // the split counters the tasks' atomics hit)
    unsigned* sync = reinterpret_cast<unsigned*>(
        (reinterpret_cast<uintptr_t>(counter + n_kv) + 127) & ~static_cast<uintptr_t>(127));
    CoreOprojArgs c{a,     d_h,     d_wo, d, q_dim, rpc, stages, used, d_h_out, sync,
                    attn_fused_mode() == 2};
    void* args[] = {&c};
    DAOP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(attn_core_oproj_kernel),
                                          dim3(sms), dim3((AT_WARPS + 1) * 32), args, smem, st));
    DAOP_CHECK_LAUNCH("attn_core_oproj");
    return DAOP_OK;
  }
  {
    static const int core_pdl = [] {
      const char* v = getenv("DAOP_ATTN_CORE_PDL");
      return v ? atoi(v) : 1;
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_kv, used);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = core_pdl ? 1 : 0;
    DAOP_CUDA(cudaLaunchKernelEx(&cfg, attn_decode_kernel, a));
    DAOP_CHECK_LAUNCH("attn_decode");
  }
  {
    const int rpc = (d + sms - 1) / sms;
    const int stages = AT_WARPS;  // one stage per consumer warp (see above)
    const size_t smem = static_cast<size_t>(stages) * q_dim * 2 + static_cast<size_t>(q_dim) * 2 +
                        2 * stages * 8;
    DAOP_CUDA(cudaFuncSetAttribute(attn_oproj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    static const int oproj_pdl = [] {
      const char* v = getenv("DAOP_ATTN_OPROJ_PDL");
      return v ? atoi(v) : 1;
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3((AT_WARPS + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = oproj_pdl ? 1 : 0;
    DAOP_CUDA(cudaLaunchKernelEx(&cfg, attn_oproj_kernel, d_h, static_cast<const uint16_t*>(o), d_wo,
                                 d, q_dim, rpc, stages, d_h_out));
    DAOP_CHECK_LAUNCH("attn_oproj");
  }
  return DAOP_OK;
}

extern "C" int daop_l2_prefetch(const void* d_p0, int64_t n0, const void* d_p1, int64_t n1,
                                daop_stream_t stream) {
  if (n0 < 0 || n1 < 0 || (n0 % 16) || (n1 % 16) ||
      (reinterpret_cast<uintptr_t>(d_p0) % 16) || (reinterpret_cast<uintptr_t>(d_p1) % 16)) {
    set_error("l2_prefetch: ranges must be 16-byte aligned multiples of 16 bytes");
    return DAOP_ERR_UNSUPPORTED;
  }
  if (n0 + n1 == 0) return DAOP_OK;
  l2_prefetch_kernel<<<sm_count(), 32, 0, as_stream(stream)>>>(
      static_cast<const uint8_t*>(d_p0), n0, static_cast<const uint8_t*>(d_p1), n1);
  DAOP_CHECK_LAUNCH("l2_prefetch");
  return DAOP_OK;
}

extern "C" int daop_set_attn_fused(int32_t fused) {
  g_attn_fused = fused < 0 ? 0 : fused > 2 ? 2 : fused;
  return DAOP_OK;
}

// profiling aid: enable != 0 zeroes and turns on the decode attention kernels'
// per-CTA global-timer stamps; h_out (3 x 256 x 2 u64, optional) receives
// them: [qkv, core, oproj][cta][start, end] of each kernel's last launch (ns)
extern "C" int daop_attn_timeline(int32_t enable, uint64_t* h_out) {
  if (h_out) DAOP_CUDA(cudaMemcpyFromSymbol(h_out, g_attn_tl, sizeof(g_attn_tl)));
  if (enable) {
    static unsigned long long zeros[3][AT_TL_CTAS][2];
    DAOP_CUDA(cudaMemcpyToSymbol(g_attn_tl, zeros, sizeof(zeros)));
  }
  DAOP_CUDA(cudaMemcpyToSymbol(g_attn_tl_on, &enable, sizeof(int)));
  return DAOP_OK;
}
