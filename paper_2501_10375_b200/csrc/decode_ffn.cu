// Decode MoE layer for one token: fused router + DAOP decision + HBM-streaming
// SwiGLU expert GEMV + combine, in ONE persistent launch.
//
//   phase 0 (every CTA, redundant & bit-identical):
//       x = bf16(rmsnorm(h) * gamma); z = x . Wg_l^T; p = softmax(z)
//       selection: mode TRUE -> top-k(p)                   (l < start / fiddler)
//                  mode PLAN -> top-k(pred_prev) + graceful degradation over
//                               the layer's HBM residence   (DAOP l >= start,
//                               policies.py:299-336 via decide.cuh)
//       CTAs 0..E-1 also compute one row each of the next-layer gate
//       (x . Wg_{l+1}^T -> p_pred) from the same x.
//   phase 1: W1/W3 rows of every resident (fast) pick, streamed HBM -> smem
//       by per-warp cp.async.bulk rings, dot with x, act = bf16(silu(g)*u).
//   grid barrier -- every warp's ring is already streaming its first W2
//       pieces while it waits, so the phase boundary does not drain HBM.
//   phase 2: W2 rows (dot with act in smem) -> y[q, r]; the warp (or the last
//       of the warps sharing a row) writes h'[r] = h[r] + sum_q w_q y[q, r]
//       in fixed q order.
//
// Bytes per call (Mixtral-8x7B, 2 resident picks): 2 x 3 x 4096 x 14336 x 2 B
// of weights + 2 x 8 x 4096 x 2 B of gates = 704,774,144 B -> HBM roofline.
#include <cooperative_groups.h>

#include "common.cuh"
#include "decide.cuh"

namespace daop {

constexpr int DW = 8;          // consumer warps per CTA, each with its own ring
constexpr int DS = 2;          // ring stages per warp
constexpr int DSB = 8192;      // bytes per stage (max piece)
constexpr int DK_MAX = 8;      // max top-k
constexpr int DE_MAX = 64;     // max experts
constexpr int D_THREADS = DW * 32;

struct DecodeArgs {
  const float* h;          // (d) fp32 residual in
  const uint16_t* gamma;   // (d) RMSNorm weight
  const uint16_t* wg;      // (E, d) gate of this layer
  const uint16_t* wg_next; // (E, d) gate of layer l+1 or null
  const float* pred_prev;  // (E) prediction carried on layer l-1 (PLAN mode)
  const uint8_t* fast_row; // (E) residence of this layer's experts
  const int32_t* slot_of;  // (E) HBM slot of expert e (valid where fast)
  const uint16_t* slab;    // expert slot slab
  int64_t slot_stride;     // elements per slot: [W1 | W3 | W2]
  int d, ffn, E, k;
  int mode;                // 0 TRUE, 1 PLAN
  int graceful;
  int weights_from_pred;   // combine weights from pred_prev (PLAN) instead of p
  float eps;
  // outputs
  uint16_t* x_out;         // (d) bf16 normalised input (stale input for layer l+1)
  float* p_true;           // (E)
  float* p_pred;           // (E) or null
  int32_t* sel;            // (k)
  float* w;                // (k)
  uint8_t* is_fast;        // (k)
  int32_t* deg;            // (2k): drop[k], sub[k]; deg[2k] = count
  float* y;                // (k, d) per-pick expert outputs
  float* h_out;            // (d) combined residual (written when every pick is fast)
  // workspace (zero-initialised once by the caller, self-resetting)
  unsigned* sync;          // [0] arrive, [1] generation, [2..2+d) per-row counters
  float* pred_logits;      // (E)
  uint16_t* act;           // (k, ffn) bf16 SwiGLU activations
};

struct DecodeSmem {
  uint64_t bar[DW][DS];
  uint64_t act_bar;
  float red[DW];
  float z[DE_MAX];
  float p[DE_MAX];
  float wsel[DK_MAX];
  int sel[DK_MAX];
  int exec_q[DK_MAX];      // pick index of the q-th executed (fast) pick
  int n_exec;
  int done1;
  float rscale;
};

struct PieceMap {
  const uint16_t* base[DK_MAX];  // slot base of executed pick
  int n_exec, d, ffn;
  int npc1, pe1;  // pieces per W1/W3 row, elements per piece
  int npc2, pe2;  // pieces per W2 row
  int64_t u1a, u1b, u2a, u2b;  // unit ranges of this warp
  int64_t n1, n;               // piece counts (phase 1, total)
};

// piece p of this warp -> source pointer, element count, vector offset
__device__ __forceinline__ void piece_at(const PieceMap& m, int64_t p, const uint16_t*& src,
                                         int& elems, int& voff) {
  if (p < m.n1) {
    const int64_t u = m.u1a + p / (2 * m.npc1);
    const int q = static_cast<int>(p % (2 * m.npc1));
    const int which = q / m.npc1, c = q % m.npc1;
    const int j = static_cast<int>(u / m.ffn);
    const int64_t i = u % m.ffn;
    voff = c * m.pe1;
    elems = min(m.pe1, m.d - voff);
    src = m.base[j] + (static_cast<int64_t>(which) * m.ffn + i) * m.d + voff;
  } else {
    const int64_t p2 = p - m.n1;
    const int64_t u = m.u2a + p2 / m.npc2;
    const int c = static_cast<int>(p2 % m.npc2);
    const int64_t r = u / m.n_exec;
    const int j = static_cast<int>(u % m.n_exec);
    voff = c * m.pe2;
    elems = min(m.pe2, m.ffn - voff);
    src = m.base[j] + 2ll * m.ffn * m.d + r * m.ffn + voff;
  }
}

__device__ __forceinline__ float dot_piece(const uint4* wp, const uint4* vp, int n16, int lane,
                                           float acc) {
#pragma unroll 4
  for (int c = lane; c < n16; c += 32) acc = dot8(wp[c], vp[c], acc);
  return acc;
}

__device__ __forceinline__ void grid_barrier(unsigned* sync, unsigned nblocks) {
  const unsigned gen = ld_acquire_gpu(sync + 1);
  __threadfence();
  const unsigned ticket = atom_add_acq_rel_gpu(sync, 1u);
  if (ticket == nblocks - 1) {
    sync[0] = 0;
    st_release_gpu(sync + 1, gen + 1);
  } else {
    while (ld_acquire_gpu(sync + 1) == gen) __nanosleep(64);
  }
}

__global__ void __launch_bounds__(D_THREADS, 1) decode_layer_kernel(DecodeArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;                                              // DW*DS*DSB
  uint16_t* act_s = reinterpret_cast<uint16_t*>(smem + DW * DS * DSB);  // k*ffn
  uint16_t* x_s = act_s + static_cast<size_t>(a.k) * a.ffn;             // d
  DecodeSmem& s = *reinterpret_cast<DecodeSmem*>(
      reinterpret_cast<uint8_t*>(x_s) + ((static_cast<size_t>(a.d) * 2 + 127) / 128) * 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = a.d, E = a.E, k = a.k;

  if (threadIdx.x == 0) {
    for (int w = 0; w < DW; ++w)
      for (int q = 0; q < DS; ++q) mbar_init(&s.bar[w][q], 1);
    mbar_init(&s.act_bar, 1);
    fence_mbar_init();
    s.done1 = 0;
  }
  // ---------------------------------------------------------------- phase 0
  // RMSNorm: x = bf16(h * rsqrt(mean(h^2) + eps) * gamma)
  float ss = 0.f;
  const float4* h4 = reinterpret_cast<const float4*>(a.h);
  for (int i = threadIdx.x; i < d / 4; i += D_THREADS) {
    const float4 v = h4[i];
    ss = fmaf(v.x, v.x, ss); ss = fmaf(v.y, v.y, ss); ss = fmaf(v.z, v.z, ss); ss = fmaf(v.w, v.w, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) s.red[warp] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < DW; ++w) t += s.red[w];
    s.rscale = 1.0f / sqrtf(t / static_cast<float>(d) + a.eps);
  }
  __syncthreads();
  const float r = s.rscale;
  for (int i = threadIdx.x; i < d / 2; i += D_THREADS) {
    const float2 hv = reinterpret_cast<const float2*>(a.h)[i];
    const uint32_t gw = reinterpret_cast<const uint32_t*>(a.gamma)[i];
    const uint32_t lo = f32_to_bf16_bits(__fmul_rn(__fmul_rn(hv.x, r), bf16lo(gw)));
    const uint32_t hi = f32_to_bf16_bits(__fmul_rn(__fmul_rn(hv.y, r), bf16hi(gw)));
    reinterpret_cast<uint32_t*>(x_s)[i] = lo | (hi << 16);
  }
  __syncthreads();
  if (blockIdx.x == 0 && a.x_out)
    for (int i = threadIdx.x; i < d / 8; i += D_THREADS)
      reinterpret_cast<uint4*>(a.x_out)[i] = reinterpret_cast<const uint4*>(x_s)[i];
  // gate logits of this layer (warp per row) + one next-layer row per CTA < E
  const int n16 = d / 8;
  for (int e = warp; e < E; e += DW) {
    const float acc = dot_piece(reinterpret_cast<const uint4*>(a.wg + static_cast<size_t>(e) * d),
                                reinterpret_cast<const uint4*>(x_s), n16, lane, 0.f);
    const float z = warp_sum(acc);
    if (lane == 0) s.z[e] = z;
  }
  if (a.wg_next && blockIdx.x < static_cast<unsigned>(E) && warp == DW - 1) {
    const int e = blockIdx.x;
    const float acc = dot_piece(
        reinterpret_cast<const uint4*>(a.wg_next + static_cast<size_t>(e) * d),
        reinterpret_cast<const uint4*>(x_s), n16, lane, 0.f);
    const float z = warp_sum(acc);
    if (lane == 0) a.pred_logits[e] = z;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = s.z[0];
    for (int i = 1; i < E; ++i) m = fmaxf(m, s.z[i]);
    float sum = 0.f;
    for (int i = 0; i < E; ++i) {
      s.p[i] = expf(s.z[i] - m);
      sum += s.p[i];
    }
    for (int i = 0; i < E; ++i) s.p[i] = s.p[i] / sum;
    int sel[DK_MAX], drop[DK_MAX], sub[DK_MAX];
    uint8_t fast[DK_MAX];
    int nd = plan_layer(a.mode ? 1 : 0, s.p, a.pred_prev, a.mode == 1, a.fast_row, E, k, 1,
                        a.mode == 1, a.graceful != 0, sel, fast, drop, sub);
    const float* wsrc = (a.mode == 1 && a.weights_from_pred) ? a.pred_prev : s.p;
    float den = 0.f;
    for (int q = 0; q < k; ++q) den += wsrc[sel[q]];
    int ne = 0;
    for (int q = 0; q < k; ++q) {
      s.sel[q] = sel[q];
      s.wsel[q] = wsrc[sel[q]] / den;
      if (fast[q]) s.exec_q[ne++] = q;
    }
    s.n_exec = ne;
    if (blockIdx.x == 0) {
      for (int i = 0; i < E; ++i) a.p_true[i] = s.p[i];
      for (int q = 0; q < k; ++q) {
        a.sel[q] = sel[q];
        a.w[q] = s.wsel[q];
        a.is_fast[q] = fast[q];
        a.deg[q] = q < nd ? drop[q] : -1;
        a.deg[k + q] = q < nd ? sub[q] : -1;
      }
      a.deg[2 * k] = nd;
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- streaming
  PieceMap m;
  m.n_exec = s.n_exec;
  m.d = d;
  m.ffn = a.ffn;
  for (int q = 0; q < m.n_exec; ++q)
    m.base[q] = a.slab + static_cast<int64_t>(a.slot_of[s.sel[s.exec_q[q]]]) * a.slot_stride;
  m.npc1 = (d * 2 + DSB - 1) / DSB;
  m.pe1 = (((d + m.npc1 - 1) / m.npc1) + 7) / 8 * 8;
  m.npc2 = (a.ffn * 2 + DSB - 1) / DSB;
  m.pe2 = (((a.ffn + m.npc2 - 1) / m.npc2) + 7) / 8 * 8;
  const int64_t W = static_cast<int64_t>(gridDim.x) * DW;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * DW + warp;
  const int64_t U1 = static_cast<int64_t>(m.n_exec) * a.ffn;
  const int64_t U2 = static_cast<int64_t>(m.n_exec) * d;
  m.u1a = U1 * gw / W;
  m.u1b = U1 * (gw + 1) / W;
  m.u2a = U2 * gw / W;
  m.u2b = U2 * (gw + 1) / W;
  m.n1 = (m.u1b - m.u1a) * 2 * m.npc1;
  m.n = m.n1 + (m.u2b - m.u2a) * m.npc2;
  const bool all_fast = m.n_exec == k;

  uint8_t* my_ring = ring + warp * DS * DSB;
  const uint64_t pol = l2_evict_first_policy();
  int64_t issued = 0;  // warp-uniform: next piece to issue
  auto issue_next = [&]() {
    if (issued < m.n) {
      if (lane == 0) {
        const uint16_t* src;
        int elems, voff;
        piece_at(m, issued, src, elems, voff);
        uint64_t* bar = &s.bar[warp][issued % DS];
        mbar_arrive_expect_tx(bar, elems * 2);
        bulk_g2s(my_ring + (issued % DS) * DSB, src, elems * 2, bar, pol);
      }
      ++issued;
    }
  };
  for (int q = 0; q < DS; ++q) issue_next();

  bool reported = false;
  auto finish_phase1 = [&]() {
    // every warp reports once; the CTA's last reporter runs the grid barrier
    // and pulls the activations into shared memory for phase 2
    reported = true;
    if (lane == 0) {
      __threadfence();
      const int old = atomicAdd(&s.done1, 1);
      if (old == DW - 1) {
        grid_barrier(a.sync, gridDim.x);
        if (blockIdx.x == 0 && a.p_pred) {  // next-layer prediction probabilities
          float z[DE_MAX], mx = -INFINITY, sum = 0.f;
          for (int i = 0; i < E; ++i) {
            z[i] = __ldcg(a.pred_logits + i);
            mx = fmaxf(mx, z[i]);
          }
          for (int i = 0; i < E; ++i) {
            z[i] = expf(z[i] - mx);
            sum += z[i];
          }
          for (int i = 0; i < E; ++i) a.p_pred[i] = z[i] / sum;
        }
        asm volatile("fence.proxy.async;" ::: "memory");
        const uint32_t bytes = static_cast<uint32_t>(m.n_exec) * a.ffn * 2;
        if (bytes == 0) {
          mbar_arrive(&s.act_bar);
        } else {
          mbar_arrive_expect_tx(&s.act_bar, bytes);
          for (int q = 0; q < m.n_exec; ++q)
            bulk_g2s_plain(act_s + static_cast<size_t>(q) * a.ffn,
                           a.act + static_cast<size_t>(s.exec_q[q]) * a.ffn, a.ffn * 2,
                           &s.act_bar);
        }
      }
    }
    __syncwarp();
  };

  float acc0 = 0.f, acc1 = 0.f;
  float yrow[DK_MAX];
  for (int64_t p = 0; p < m.n; ++p) {
    if (p == m.n1) {
      if (!reported) finish_phase1();
      mbar_wait(&s.act_bar, 0);
    }
    const int stg = static_cast<int>(p % DS);
    mbar_wait(&s.bar[warp][stg], static_cast<uint32_t>((p / DS) & 1));
    const uint16_t* src;
    int elems, voff;
    piece_at(m, p, src, elems, voff);
    const uint4* wp = reinterpret_cast<const uint4*>(my_ring + stg * DSB);
    if (p < m.n1) {
      const int q = static_cast<int>(p % (2 * m.npc1));
      const float part = dot_piece(wp, reinterpret_cast<const uint4*>(x_s + voff), elems / 8,
                                   lane, 0.f);
      if (q < m.npc1) acc0 += part; else acc1 += part;
      __syncwarp();
      issue_next();  // refill the stage we just drained
      if (q == 2 * m.npc1 - 1) {  // end of a (W1 row, W3 row) pair
        const float g = warp_sum(acc0), u = warp_sum(acc1);
        acc0 = acc1 = 0.f;
        if (lane == 0) {
          const int64_t unit = m.u1a + p / (2 * m.npc1);
          const int j = static_cast<int>(unit / a.ffn);
          const int64_t i = unit % a.ffn;
          a.act[static_cast<int64_t>(s.exec_q[j]) * a.ffn + i] = f32_to_bf16_bits(silu_f32(g) * u);
        }
      }
    } else {
      const int64_t p2 = p - m.n1;
      const int64_t unit = m.u2a + p2 / m.npc2;
      const int c = static_cast<int>(p2 % m.npc2);
      const int j = static_cast<int>(unit % m.n_exec);
      acc0 = dot_piece(wp, reinterpret_cast<const uint4*>(act_s + static_cast<size_t>(j) * a.ffn + voff),
                       elems / 8, lane, acc0);
      __syncwarp();
      issue_next();
      if (c == m.npc2 - 1) {  // end of the (row, pick) unit
        const float yv = warp_sum(acc0);
        acc0 = 0.f;
        const int64_t row = unit / m.n_exec;
        yrow[j] = yv;
        if (lane == 0) a.y[static_cast<int64_t>(s.exec_q[j]) * d + row] = yv;
        if (all_fast) {
          const int64_t first = row * m.n_exec, last = first + m.n_exec - 1;
          const bool whole = first >= m.u2a && last < m.u2b;
          if (whole) {
            if (j == m.n_exec - 1 && lane == 0) {  // whole row is ours: combine in registers
              float o = a.h[row];
              for (int q = 0; q < k; ++q) o = fmaf(s.wsel[q], yrow[q], o);
              a.h_out[row] = o;
            }
          } else if (unit == last || unit == m.u2b - 1) {
            // row shared with a neighbouring warp: the last arriver combines
            if (lane == 0) {
              const int64_t lo = first > m.u2a ? first : m.u2a;
              const unsigned mine = static_cast<unsigned>(unit - lo + 1);
              __threadfence();
              const unsigned old = atomicAdd(a.sync + 2 + row, mine);
              if (old + mine == static_cast<unsigned>(m.n_exec)) {
                __threadfence();
                float o = a.h[row];
                for (int q = 0; q < k; ++q)
                  o = fmaf(s.wsel[q], __ldcg(a.y + static_cast<int64_t>(q) * d + row), o);
                a.h_out[row] = o;
                a.sync[2 + row] = 0;
              }
            }
          }
        }
      }
    }
  }
  if (!reported) finish_phase1();
}

}  // namespace daop

using namespace daop;

extern "C" int daop_decode_workspace(int32_t d, int32_t ffn, int32_t E, int32_t k,
                                     int64_t* bytes) {
  // sync counters (2 + d uint32) | pred logits (E f32) | act (k*ffn bf16)
  *bytes = ((2 + static_cast<int64_t>(d)) * 4 + 255) / 256 * 256 + 256 +
           (static_cast<int64_t>(k) * ffn * 2 + 255) / 256 * 256;
  return DAOP_OK;
}

extern "C" int daop_decode_layer(const float* h, const uint16_t* gamma, const uint16_t* wg,
                                 const uint16_t* wg_next, const float* pred_prev,
                                 const uint8_t* fast_row, const int32_t* slot_of,
                                 const uint16_t* slab, int64_t slot_stride, int32_t d,
                                 int32_t ffn, int32_t E, int32_t k, int32_t mode,
                                 int32_t graceful, int32_t weights_from_pred, float eps,
                                 uint16_t* x_out, float* p_true, float* p_pred, int32_t* sel,
                                 float* w, uint8_t* is_fast, int32_t* deg, float* y,
                                 float* h_out, void* workspace, int32_t grid,
                                 daop_stream_t stream) {
  if (E < 2 || E > DE_MAX || k < 1 || k > DK_MAX || k > E || d % 8 || ffn % 8) {
    set_error("decode_layer: unsupported shape (E=%d k=%d d=%d ffn=%d)", E, k, d, ffn);
    return DAOP_ERR_UNSUPPORTED;
  }
  if (mode == 1 && !pred_prev) {
    set_error("decode_layer: PLAN mode needs the previous layer's prediction");
    return DAOP_ERR_PREDICTION_MISSING;
  }
  DecodeArgs a;
  a.h = h; a.gamma = gamma; a.wg = wg; a.wg_next = wg_next; a.pred_prev = pred_prev;
  a.fast_row = fast_row; a.slot_of = slot_of; a.slab = slab; a.slot_stride = slot_stride;
  a.d = d; a.ffn = ffn; a.E = E; a.k = k; a.mode = mode; a.graceful = graceful;
  a.weights_from_pred = weights_from_pred; a.eps = eps;
  a.x_out = x_out; a.p_true = p_true; a.p_pred = wg_next ? p_pred : nullptr; a.sel = sel;
  a.w = w; a.is_fast = is_fast; a.deg = deg; a.y = y; a.h_out = h_out;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  a.sync = reinterpret_cast<unsigned*>(ws);
  const int64_t o1 = ((2 + static_cast<int64_t>(d)) * 4 + 255) / 256 * 256;
  a.pred_logits = reinterpret_cast<float*>(ws + o1);
  a.act = reinterpret_cast<uint16_t*>(ws + o1 + 256);

  const size_t smem = static_cast<size_t>(DW) * DS * DSB + static_cast<size_t>(k) * ffn * 2 +
                      (static_cast<size_t>(d) * 2 + 127) / 128 * 128 + sizeof(DecodeSmem) + 128;
  if (smem > 227 * 1024) {
    set_error("decode_layer: %zu B of shared memory exceeds 227 KB (k*ffn too large)", smem);
    return DAOP_ERR_UNSUPPORTED;
  }
  DAOP_CUDA(cudaFuncSetAttribute(decode_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const int sms = sm_count();
  if (grid <= 0 || grid > sms) grid = sms;
  if (grid < E) grid = E;  // CTAs 0..E-1 own one next-layer gate row each
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(D_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DAOP_CUDA(cudaLaunchKernelEx(&cfg, decode_layer_kernel, a));
  return DAOP_OK;
}
