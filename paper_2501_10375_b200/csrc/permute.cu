// Token -> expert permutation by histogram + exclusive scan, and the
// weighted combine / unpermute.
//
// Order contract (deterministic, stable): the T*k assignments (t, j) are
// sorted by (expert, t, j).  offsets[e] is the exclusive scan of the expert
// histogram; perm[p] = t*k + j of the row at sorted position p; inv[t*k+j] =
// p.  x_perm[p] = x[t] feeds the grouped GEMM's A operand through TMA.
//
//   count   : per-CTA expert histograms of contiguous assignment chunks
//   scan    : one CTA, exclusive scan over (expert, chunk) -> chunk bases
//   scatter : per chunk, stable in-chunk ranks with __match_any_sync,
//             warp totals prefix-summed in shared memory
//   gather  : one warp per sorted row, 16-byte coalesced row copy
//   combine : h'[t] = h[t] + sum_{j=0..k-1} w[t,j] * y[inv[t,j]]  (fixed j order)
#include <algorithm>

#include "common.cuh"

namespace daop {

constexpr int P_THREADS = 256;
constexpr int P_MAX_E = 256;

__global__ void perm_count_kernel(const int32_t* __restrict__ ids, int64_t n, int64_t chunk, int E,
                                  int32_t* __restrict__ counts /* [chunks][E] */) {
  pdl_prologue();  // (launched with launch_pdl)
  __shared__ int32_t h[P_MAX_E];
  for (int i = threadIdx.x; i < E; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t a = blockIdx.x * chunk, b = min(n, a + chunk);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) atomicAdd(&h[ids[i]], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) counts[blockIdx.x * (int64_t)E + i] = h[i];
}

__global__ void perm_scan_kernel(int32_t* __restrict__ counts, int nchunks, int E,
                                 int64_t* __restrict__ offsets) {
  pdl_prologue();  // (launched with launch_pdl)
  // thread e: serial scan over chunks of expert e (totals), then thread 0 scans experts
  __shared__ int64_t tot[P_MAX_E + 1];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t s = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int32_t v = counts[c * (int64_t)E + e];
      counts[c * (int64_t)E + e] = static_cast<int32_t>(s);  // in-expert base of chunk c
      s += v;
    }
    tot[e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = s;
      s += tot[e];
    }
    offsets[E] = s;
  }
}

__global__ void perm_scatter_kernel(const int32_t* __restrict__ ids, int64_t n, int64_t chunk,
                                    int E, const int32_t* __restrict__ chunk_base,
                                    const int64_t* __restrict__ offsets,
                                    int32_t* __restrict__ perm, int32_t* __restrict__ inv) {
  pdl_prologue();  // (launched with launch_pdl)
  __shared__ int32_t run[P_MAX_E];                   // running count per expert in this chunk
  __shared__ int32_t wtot[P_THREADS / 32][P_MAX_E];  // per-warp totals of the current tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < E; i += blockDim.x) run[i] = 0;
  const int64_t a = blockIdx.x * chunk, b = min(n, a + chunk);
  for (int64_t base = a; base < b; base += P_THREADS) {
    for (int i = threadIdx.x; i < (P_THREADS / 32) * E; i += blockDim.x)
      wtot[i / E][i % E] = 0;
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    const bool ok = i < b;
    const int e = ok ? ids[i] : -1 - lane;  // distinct dummies never match real ids
    const unsigned same = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(same & ((1u << lane) - 1u));
    if (ok && rank == 0) wtot[warp][e] = __popc(same);
    __syncthreads();
    if (ok) {
      int before = 0;
      for (int w = 0; w < warp; ++w) before += wtot[w][e];
      const int64_t pos = offsets[e] + chunk_base[blockIdx.x * (int64_t)E + e] + run[e] + before + rank;
      perm[pos] = static_cast<int32_t>(i);
      inv[i] = static_cast<int32_t>(pos);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < E; x += blockDim.x) {
      int s = 0;
      for (int w = 0; w < P_THREADS / 32; ++w) s += wtot[w][x];
      run[x] += s;
    }
    __syncthreads();
  }
}

// n <= one chunk (decode-sized batches, prefill up to 4096 rows): count, scan
// and the stable scatter of the three kernels above in ONE CTA -- the same
// order (rows by expert, then by i), one launch instead of three
__global__ void __launch_bounds__(P_THREADS, 1)
    perm_single_kernel(const int32_t* __restrict__ ids, int64_t n, int E,
                       int64_t* __restrict__ offsets, int32_t* __restrict__ perm,
                       int32_t* __restrict__ inv) {
  pdl_prologue();  // (launched with launch_pdl)
  __shared__ int32_t cnt[P_MAX_E];
  __shared__ int32_t run[P_MAX_E];
  __shared__ int64_t off[P_MAX_E];
  __shared__ int32_t wtot[P_THREADS / 32][P_MAX_E];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < E; i += blockDim.x) cnt[i] = run[i] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&cnt[ids[i]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int e = 0; e < E; ++e) {
      off[e] = offsets[e] = s;
      s += cnt[e];
    }
    offsets[E] = s;
  }
  for (int64_t base = 0; base < n; base += P_THREADS) {
    for (int i = threadIdx.x; i < (P_THREADS / 32) * E; i += blockDim.x) wtot[i / E][i % E] = 0;
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    const bool ok = i < n;
    const int e = ok ? ids[i] : -1 - lane;  // distinct dummies never match real ids
    const unsigned same = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(same & ((1u << lane) - 1u));
    if (ok && rank == 0) wtot[warp][e] = __popc(same);
    __syncthreads();
    if (ok) {
      int before = 0;
      for (int w = 0; w < warp; ++w) before += wtot[w][e];
      const int64_t pos = off[e] + run[e] + before + rank;
      perm[pos] = static_cast<int32_t>(i);
      inv[i] = static_cast<int32_t>(pos);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < E; x += blockDim.x) {
      int s = 0;
      for (int w = 0; w < P_THREADS / 32; ++w) s += wtot[w][x];
      run[x] += s;
    }
    __syncthreads();  // run[] complete before the next tile zeroes wtot / reads run
  }
}

// token-major gather: a warp reads token t's x row ONCE and stores it at its
// k sorted positions inv[t, j] (reading in permuted order would fetch every
// row k times, far apart in time)
template <int K>
__global__ void perm_gather_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ inv,
                                   int64_t T, int k_rt, int n16, uint4* __restrict__ x_perm) {
  pdl_prologue();  // (launched with launch_pdl)
  const int lane = threadIdx.x & 31;
  const int k = K > 0 ? K : k_rt;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < T;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint4* s = x + t * n16;
    if constexpr (K > 0) {
      uint4* d[K];
#pragma unroll
      for (int j = 0; j < K; ++j) d[j] = x_perm + static_cast<int64_t>(inv[t * K + j]) * n16;
#pragma unroll 4
      for (int c = lane; c < n16; c += 32) {
        const uint4 v = __ldcs(s + c);
#pragma unroll
        for (int j = 0; j < K; ++j) d[j][c] = v;
      }
    } else {
      for (int c = lane; c < n16; c += 32) {
        const uint4 v = __ldcs(s + c);
        for (int j = 0; j < k; ++j) x_perm[static_cast<int64_t>(inv[t * k + j]) * n16 + c] = v;
      }
    }
  }
}

// one warp per token row; the k source rows and weights are hoisted, the
// d-loop is unrolled so each lane keeps (k+1) x 4 independent 16 B loads in
// flight.  Sum order per element: h, then j = 0..k-1 (fmaf), fixed.
template <int K>
__global__ void combine_kernel(const float* __restrict__ h, const float* __restrict__ y,
                               const int32_t* __restrict__ inv, const float* __restrict__ w,
                               int64_t T, int k_rt, int d4, float* __restrict__ out) {
  pdl_prologue();  // (launched with launch_pdl)
  const int lane = threadIdx.x & 31;
  const int k = K > 0 ? K : k_rt;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < T;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float4* hr = reinterpret_cast<const float4*>(h) + t * d4;
    float4* o = reinterpret_cast<float4*>(out) + t * d4;
    if constexpr (K > 0) {
      const float4* yr[K];
      float wj[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        yr[j] = reinterpret_cast<const float4*>(y) + static_cast<int64_t>(inv[t * K + j]) * d4;
        wj[j] = w[t * K + j];
      }
#pragma unroll 4
      for (int c = lane; c < d4; c += 32) {
        float4 acc = __ldcs(hr + c);
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const float4 v = __ldcs(yr[j] + c);
          acc.x = fmaf(wj[j], v.x, acc.x);
          acc.y = fmaf(wj[j], v.y, acc.y);
          acc.z = fmaf(wj[j], v.z, acc.z);
          acc.w = fmaf(wj[j], v.w, acc.w);
        }
        __stcs(o + c, acc);
      }
    } else {
      for (int c = lane; c < d4; c += 32) {
        float4 acc = hr[c];
        for (int j = 0; j < k; ++j) {
          const float wj = w[t * k + j];
          const float4 v = reinterpret_cast<const float4*>(y)[static_cast<int64_t>(inv[t * k + j]) * d4 + c];
          acc.x = fmaf(wj, v.x, acc.x);
          acc.y = fmaf(wj, v.y, acc.y);
          acc.z = fmaf(wj, v.z, acc.z);
          acc.w = fmaf(wj, v.w, acc.w);
        }
        o[c] = acc;
      }
    }
  }
}

// ---------------------------------------------------------------- bulk-DMA pipelines
//
// Row-streaming kernels for the big prefill passes: one CTA per SM, a ring of
// shared-memory stages filled by cp.async.bulk (one DMA per row) and drained
// by cp.async.bulk stores, so each SM keeps ~200 KB in flight with a handful
// of instructions (the register-staged versions above stall on memory
// latency at ~55 % occupancy: ncu 2.5-3.4 TB/s).


// out[t] = h[t] + sum_j w[t,j] * y[inv[t,j]]  (fixed j order, fmaf: the same
// arithmetic as combine_kernel).  Stage = [h row | y rows of the k picks].
template <int K>
__global__ void __launch_bounds__(256, 1)
    combine_bulk_kernel(const float* __restrict__ h, const float* __restrict__ y,
                        const int32_t* __restrict__ inv, const float* __restrict__ w, int64_t T,
                        int d, int stages, float* __restrict__ out) {
  pdl_prologue();  // (launched with launch_pdl)
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t row = static_cast<uint32_t>(d) * 4;
  const uint32_t stage_bytes = row * (K + 1);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * stage_bytes);
  const int64_t n_my = T > blockIdx.x ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto issue = [&](int64_t i) {  // thread 0: loads of my i-th token into stage i % stages
    const int st = static_cast<int>(i % stages);
    const int64_t t = blockIdx.x + i * gridDim.x;
    uint8_t* sb = smem + static_cast<size_t>(st) * stage_bytes;
    mbar_arrive_expect_tx(&full[st], stage_bytes);
    bulk_g2s_plain(sb, h + t * d, row, &full[st]);
#pragma unroll
    for (int j = 0; j < K; ++j)
      bulk_g2s_plain(sb + (j + 1) * row, y + static_cast<int64_t>(inv[t * K + j]) * d, row,
                     &full[st]);
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < stages; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
    for (int64_t i = 0; i < n_my && i < stages; ++i) issue(i);
  }
  __syncthreads();
  for (int64_t i = 0; i < n_my; ++i) {
    const int st = static_cast<int>(i % stages);
    const int64_t t = blockIdx.x + i * gridDim.x;
    float* sb = reinterpret_cast<float*>(smem + static_cast<size_t>(st) * stage_bytes);
    mbar_wait(&full[st], static_cast<uint32_t>((i / stages) & 1));
    float wj[K];
#pragma unroll
    for (int j = 0; j < K; ++j) wj[j] = w[t * K + j];
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
      float4 acc = reinterpret_cast<const float4*>(sb)[c];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const float4 v = reinterpret_cast<const float4*>(sb + (j + 1) * d)[c];
        acc.x = fmaf(wj[j], v.x, acc.x);
        acc.y = fmaf(wj[j], v.y, acc.y);
        acc.z = fmaf(wj[j], v.z, acc.z);
        acc.w = fmaf(wj[j], v.w, acc.w);
      }
      reinterpret_cast<float4*>(sb)[c] = acc;  // result in place of h
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(out + t * d, sb, row);
      bulk_commit();
      // refill the stage stored one iteration ago (this store stays in flight)
      if (i >= 1 && i - 1 + stages < n_my) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(1) : "memory");
        issue(i - 1 + stages);
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// token-major gather with bulk DMAs: x row -> smem -> its k sorted positions
__global__ void __launch_bounds__(32, 1)
    gather_bulk_kernel(const uint16_t* __restrict__ x, const int32_t* __restrict__ inv,
                       int64_t T, int k, int d, int stages, uint16_t* __restrict__ x_perm) {
  pdl_prologue();  // (launched with launch_pdl)
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t row = static_cast<uint32_t>(d) * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(stages) * row);
  if (threadIdx.x != 0) return;
  const int64_t n_my = T > blockIdx.x ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  for (int st = 0; st < stages; ++st) mbar_init(&full[st], 1);
  fence_mbar_init();
  auto issue = [&](int64_t i) {
    const int st = static_cast<int>(i % stages);
    const int64_t t = blockIdx.x + i * gridDim.x;
    mbar_arrive_expect_tx(&full[st], row);
    bulk_g2s_plain(smem + static_cast<size_t>(st) * row, x + t * d, row, &full[st]);
  };
  // the first refill happens at iteration 1: prime stages - 1 loads plus one
  for (int64_t i = 0; i < n_my && i < stages; ++i) issue(i);
  for (int64_t i = 0; i < n_my; ++i) {
    const int st = static_cast<int>(i % stages);
    const int64_t t = blockIdx.x + i * gridDim.x;
    mbar_wait(&full[st], static_cast<uint32_t>((i / stages) & 1));
    for (int j = 0; j < k; ++j)
      bulk_s2g(x_perm + static_cast<int64_t>(inv[t * k + j]) * d,
               smem + static_cast<size_t>(st) * row, row);
    bulk_commit();
    // refill the stage stored one iteration ago (its stores have had a whole
    // iteration to read it; this one's stay in flight)
    if (i >= 1 && i - 1 + stages < n_my) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(1) : "memory");
      issue(i - 1 + stages);
    }
  }
  bulk_wait_all();
}

// small batches (decode): one CTA per token, every thread a few float4 of
// the row -- one memory round trip instead of a warp walking 16 KB
template <int K>
__global__ void combine_small_kernel(const float* __restrict__ h, const float* __restrict__ y,
                                     const int32_t* __restrict__ inv, const float* __restrict__ w,
                                     int d4, float* __restrict__ out) {
  pdl_prologue();  // (launched with launch_pdl)
  const int64_t t = blockIdx.x;
  const float4* hr = reinterpret_cast<const float4*>(h) + t * d4;
  float4* o = reinterpret_cast<float4*>(out) + t * d4;
  const float4* yr[K];
  float wj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    yr[j] = reinterpret_cast<const float4*>(y) + static_cast<int64_t>(inv[t * K + j]) * d4;
    wj[j] = w[t * K + j];
  }
  for (int c = threadIdx.x; c < d4; c += blockDim.x) {
    float4 acc = hr[c];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const float4 v = yr[j][c];
      acc.x = fmaf(wj[j], v.x, acc.x);
      acc.y = fmaf(wj[j], v.y, acc.y);
      acc.z = fmaf(wj[j], v.z, acc.z);
      acc.w = fmaf(wj[j], v.w, acc.w);
    }
    o[c] = acc;
  }
}

// small batches: one CTA per token row of x, stored at its k sorted positions
__global__ void gather_small_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ inv,
                                    int k, int n16, uint4* __restrict__ x_perm) {
  pdl_prologue();  // (launched with launch_pdl)
  const int64_t t = blockIdx.x;
  for (int c = threadIdx.x; c < n16; c += blockDim.x) {
    const uint4 v = x[t * n16 + c];
    for (int j = 0; j < k; ++j) x_perm[static_cast<int64_t>(inv[t * k + j]) * n16 + c] = v;
  }
}

// decode-side combine when some picks ran on the host tier:
// out[i] = h[i] + sum_{q<k} w[q] * y[q, i]   (fixed q order, like the fused path)
__global__ void combine_dense_kernel(const float* __restrict__ h, const float* __restrict__ y,
                                     const float* __restrict__ w, int k, int d,
                                     float* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
    float o = h[i];
    for (int q = 0; q < k; ++q) o = fmaf(w[q], y[static_cast<int64_t>(q) * d + i], o);
    out[i] = o;
  }
}

}  // namespace daop

using namespace daop;

// tuning (daop_set_stream_mode): gather 0 = auto (bulk DMA rows for large T),
// 1 = warp-per-token registers; combine 0 = auto (bulk), 1 = warp-per-token
static int g_gather_variant = 0, g_combine_variant = 0;
static int g_bulk_ctas_per_sm = 2, g_combine_stages = 4;  // profiles/r02/stream_kernels.json

extern "C" {

int daop_set_stream_mode(int32_t gather, int32_t combine, int32_t gather_ctas_per_sm,
                         int32_t combine_stages) {
  g_gather_variant = gather;
  g_combine_variant = combine;
  if (gather_ctas_per_sm > 0) g_bulk_ctas_per_sm = gather_ctas_per_sm;
  if (combine_stages > 0) g_combine_stages = combine_stages;
  return DAOP_OK;
}

int daop_permute_workspace(int64_t T, int32_t k, int32_t E, int64_t* bytes) {
  const int64_t n = T * k;
  int64_t chunks = (n + 4095) / 4096;
  if (chunks < 1) chunks = 1;
  *bytes = chunks * E * 4 + 256;
  return DAOP_OK;
}

int daop_permute(const int32_t* ids, int64_t T, int32_t k, int32_t E, const uint16_t* x, int32_t d,
                 int64_t* offsets, int32_t* perm, int32_t* inv, uint16_t* x_perm,
                 void* workspace, int64_t ws_bytes, daop_stream_t stream) {
  if (E < 1 || E > P_MAX_E || k < 1 || (x_perm && d % 8 != 0)) {
    set_error("permute: unsupported (E=%d, k=%d, d=%d)", E, k, d);
    return DAOP_ERR_UNSUPPORTED;
  }
  const int64_t n = T * k;
  int64_t need = 0;
  daop_permute_workspace(T, k, E, &need);
  if (ws_bytes < need) {
    set_error("permute: workspace %lld < %lld bytes", (long long)ws_bytes, (long long)need);
    return DAOP_ERR_SHAPE;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t chunk = 4096;
  int nchunks = static_cast<int>((n + chunk - 1) / chunk);
  if (nchunks < 1) nchunks = 1;
  int32_t* counts = static_cast<int32_t*>(workspace);
  if (nchunks == 1) {
    DAOP_CUDA(launch_pdl(perm_single_kernel, dim3(1), dim3(P_THREADS), 0, st, ids, n, E, offsets, perm, inv));
  } else {
    DAOP_CUDA(launch_pdl(perm_count_kernel, dim3(nchunks), dim3(P_THREADS), 0, st, ids, n, chunk, E, counts));
    DAOP_CUDA(launch_pdl(perm_scan_kernel, dim3(1), dim3(256), 0, st, counts, nchunks, E, offsets));
    DAOP_CUDA(launch_pdl(perm_scatter_kernel, dim3(nchunks), dim3(P_THREADS), 0, st, ids, n, chunk, E, counts, offsets, perm,
                                                       inv));
  }
  DAOP_CHECK_LAUNCH("permute");
  if (x_perm && n > 0) {
    int64_t blocks = (T * 32 + 255) / 256;
    const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
    if (blocks > cap) blocks = cap;
    const uint4* xs = reinterpret_cast<const uint4*>(x);
    uint4* xp = reinterpret_cast<uint4*>(x_perm);
    const size_t row = static_cast<size_t>(d) * 2;
    if (T < 2 * sm_count()) {  // decode-sized batches
      DAOP_CUDA(launch_pdl(gather_small_kernel, dim3(static_cast<int>(T)), dim3(256), 0, st, xs, inv, k, d / 8, xp));
    } else if (g_gather_variant == 0 && T >= 4 * sm_count() && row % 16 == 0 && row <= 16 * 1024) {
      const int stages = static_cast<int>(std::min<size_t>(16, (48 * 1024) / row));
      const size_t smem = row * stages + 16 * 8 + 64;
      DAOP_CUDA(cudaFuncSetAttribute(gather_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      DAOP_CUDA(launch_pdl(gather_bulk_kernel, dim3(g_bulk_ctas_per_sm * sm_count()), dim3(32), smem, st, x, inv, T, k, d,
                                                                         stages, x_perm));
    } else if (k == 2)
      DAOP_CUDA(launch_pdl(perm_gather_kernel<2>, dim3(static_cast<int>(blocks)), dim3(256), 0, st, xs, inv, T, k, d / 8, xp));
    else
      DAOP_CUDA(launch_pdl(perm_gather_kernel<0>, dim3(static_cast<int>(blocks)), dim3(256), 0, st, xs, inv, T, k, d / 8, xp));
    DAOP_CHECK_LAUNCH("permute_gather");
  }
  return DAOP_OK;
}

int daop_combine(const float* h, const float* y_sorted, const int32_t* inv, const float* w,
                 int64_t T, int32_t k, int32_t d, float* out, daop_stream_t stream) {
  if (d % 4 != 0) {
    set_error("combine: d must be a multiple of 4");
    return DAOP_ERR_UNSUPPORTED;
  }
  if (T == 0) return DAOP_OK;
  int64_t blocks = (T * 32 + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  auto launch = [&](auto kern) -> cudaError_t {
    return launch_pdl(kern, dim3(static_cast<int>(blocks)), dim3(256), 0, as_stream(stream), h,
                      y_sorted, inv, w, T, k, d / 4, out);
  };
  if (k == 2 && T < 2 * sm_count()) {  // decode-sized batches
    DAOP_CUDA(launch_pdl(combine_small_kernel<2>, dim3(static_cast<int>(T)), dim3(256), 0, as_stream(stream), 
        h, y_sorted, inv, w, d / 4, out));
    DAOP_CHECK_LAUNCH("combine_small");
    return DAOP_OK;
  }
  if (g_combine_variant == 0 && k == 2 && d % 4 == 0 && T >= sm_count()) {
    const size_t stage = static_cast<size_t>(d) * 4 * 3;
    const int stages = static_cast<int>(std::min<size_t>(g_combine_stages, (200 * 1024) / stage));
    if (stages >= 2) {
      const size_t smem = stage * stages + 64;
      DAOP_CUDA(cudaFuncSetAttribute(combine_bulk_kernel<2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      DAOP_CUDA(launch_pdl(combine_bulk_kernel<2>, dim3(sm_count()), dim3(256), smem, as_stream(stream), 
          h, y_sorted, inv, w, T, d, stages, out));
      DAOP_CHECK_LAUNCH("combine_bulk");
      return DAOP_OK;
    }
  }
  if (k == 1) DAOP_CUDA(launch(combine_kernel<1>));
  else if (k == 2) DAOP_CUDA(launch(combine_kernel<2>));
  else if (k == 4) DAOP_CUDA(launch(combine_kernel<4>));
  else DAOP_CUDA(launch(combine_kernel<0>));
  DAOP_CHECK_LAUNCH("combine");
  return DAOP_OK;
}

int daop_combine_dense(const float* h, const float* y, const float* w, int32_t k, int32_t d,
                       float* out, daop_stream_t stream) {
  combine_dense_kernel<<<(d + 255) / 256, 256, 0, as_stream(stream)>>>(h, y, w, k, d, out);
  DAOP_CHECK_LAUNCH("combine_dense");
  return DAOP_OK;
}

}  // extern "C"
