// Expert-parallel dispatch / combine over NVLink peer memory.
//
// Every rank owns one symmetric workspace (same layout on every GPU, opened
// by the peers through CUDA IPC) and the device table `peers[G]` of the G
// workspace base addresses as seen from this GPU (peers[rank] = its own).
// One MoE layer, all on the rank's stream, no host synchronisation:
//
//   publish  : per-expert row counts of this rank's permutation -> counts
//              slot [epoch&1][rank] of EVERY peer, then flag counts[rank]
//   dispatch : wait for all G count flags; every rank derives the same
//              expert-major receive layout (expert, then source rank) from
//              the G x E count matrix; a warp per permuted row gathers the
//              token's bf16 x row and stores it straight into the owner's
//              receive buffer (remote NVLink stores: the permutation gather
//              and the all-to-all are one pass); the last CTA flags x[rank]
//              on every peer
//   recv     : wait for the G x flags; local expert offsets (for the grouped
//              GEMMs) and the per-row return address table (source rank's
//              y_back + its permuted row) from the count matrix
//   experts  : tcgen05 grouped up GEMM on the receive buffer, then the down
//              GEMM whose epilogue stores every fp32 output row through the
//              return table -- straight into the source rank's y_back over
//              NVLink, tile by tile as the MMAs finish -- and whose last CTA
//              flags y[rank] on every peer (grouped_gemm.cu, EpSignal)
//   back     : wait for the G y flags; the fixed-order combine kernel reads
//              y_back in permuted order (unchanged single-GPU combine)
//
// Flags carry a monotonically increasing epoch (one per layer call), so
// they never need resetting; the count slots are double-buffered by epoch
// parity.  A peer can run at most one phase ahead (it needs this rank's
// outputs to finish its own layer), which is what makes the single receive /
// y_back buffers and the two count slots sufficient.  Spins time out (20 s)
// into an error flag instead of hanging the GPU.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ep.cuh"

namespace daop {

static inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint8_t* ws_of(const uint64_t* peers, int s) {
  return reinterpret_cast<uint8_t*>(peers[s]);
}

// wait until flag[s] has reached `epoch` for every s < G (wrap-safe compare);
// false (and the error flag set) on timeout
__device__ bool ep_wait_flags(const uint8_t* ws, int64_t flags_off, int G, unsigned epoch) {
  const unsigned* f = reinterpret_cast<const unsigned*>(ws + flags_off);
  const unsigned long long t0 = global_ns();
  for (int s = 0; s < G; ++s) {
    while (static_cast<int>(ld_acquire_sys(f + s) - epoch) < 0) {
      if (global_ns() - t0 > EP_TIMEOUT_NS) {
        atomicExch(reinterpret_cast<unsigned*>(const_cast<uint8_t*>(ws) + EP_ERR), 1u);
        return false;
      }
      __nanosleep(100);
    }
  }
  return true;
}

__device__ __forceinline__ const int64_t* ep_counts(const uint8_t* ws, unsigned epoch) {
  return reinterpret_cast<const int64_t*>(ws + EP_COUNTS) + (epoch & 1) * EP_MAX_G * EP_MAX_E;
}

// ---------------------------------------------------------------- publish

__global__ void ep_publish_kernel(const uint64_t* peers, int rank, int G, int E,
                                  const int64_t* offsets, unsigned epoch) {
  const int e = threadIdx.x;
  if (e < E) {
    const int64_t c = offsets[e + 1] - offsets[e];
    for (int s = 0; s < G; ++s) {
      int64_t* dst = reinterpret_cast<int64_t*>(ws_of(peers, s) + EP_COUNTS) +
                     (epoch & 1) * EP_MAX_G * EP_MAX_E + rank * EP_MAX_E + e;
      *reinterpret_cast<volatile int64_t*>(dst) = c;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < G; ++s)
      st_release_sys(reinterpret_cast<unsigned*>(ws_of(peers, s) + EP_FLAGS_COUNTS) + rank, epoch);
}

// ---------------------------------------------------------------- dispatch

struct EpLayout {  // derived from the G x E count matrix (identical on every rank)
  int64_t own_off[EP_MAX_E + 1];  // this rank's permuted offsets
  int64_t dst_row[EP_MAX_E];      // first receive row of (this rank, e) at owner(e)
};

__device__ void ep_layout(const int64_t* cnt, int rank, int G, int E, EpLayout& L) {
  // single thread
  int64_t acc = 0;
  for (int e = 0; e < E; ++e) {
    L.own_off[e] = acc;
    acc += cnt[rank * EP_MAX_E + e];
  }
  L.own_off[E] = acc;
  for (int e = 0; e < E; ++e) {
    const int o = e * G / E;
    int64_t base = 0;
    for (int e2 = 0; e2 < e; ++e2)
      if (e2 * G / E == o)
        for (int s = 0; s < G; ++s) base += cnt[s * EP_MAX_E + e2];
    for (int s = 0; s < rank; ++s) base += cnt[s * EP_MAX_E + e];
    L.dst_row[e] = base;
  }
}

constexpr int EP_WARPS = 8;

__global__ void __launch_bounds__(EP_WARPS * 32)
    ep_dispatch_kernel(const uint64_t* peers, int rank, int G, int E, int k, int d,
                       const uint16_t* x, const int32_t* perm, int64_t recv_off,
                       unsigned epoch) {
  __shared__ EpLayout L;
  __shared__ int ok;
  uint8_t* me = ws_of(peers, rank);
  if (threadIdx.x == 0) {
    ok = ep_wait_flags(me, EP_FLAGS_COUNTS, G, epoch);
    if (ok) ep_layout(ep_counts(me, epoch), rank, G, E, L);
  }
  __syncthreads();
  if (ok) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t rows = L.own_off[E];
    const int n16 = d / 8;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * EP_WARPS + warp; i < rows;
         i += static_cast<int64_t>(gridDim.x) * EP_WARPS) {
      int e = 0;
      while (L.own_off[e + 1] <= i) ++e;
      const int o = e * G / E;
      const int64_t t = perm[i] / k;
      const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
      uint4* dst = reinterpret_cast<uint4*>(ws_of(peers, o) + recv_off) +
                   (L.dst_row[e] + (i - L.own_off[e])) * n16;
#pragma unroll 8
      for (int c = lane; c < n16; c += 32) dst[c] = __ldg(src + c);
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* done = reinterpret_cast<unsigned*>(me + EP_DONE_DISPATCH);
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0;
      __threadfence_system();
      for (int s = 0; s < G; ++s)
        st_release_sys(reinterpret_cast<unsigned*>(ws_of(peers, s) + EP_FLAGS_X) + rank, epoch);
    }
  }
}

// ---------------------------------------------------------------- receive side

__global__ void ep_recv_kernel(const uint64_t* peers, int rank, int G, int E, int d,
                               int64_t yback_off, unsigned epoch) {
  __shared__ int64_t lo[EP_MAX_E + 1];
  __shared__ int64_t cnt[EP_MAX_G * EP_MAX_E];
  __shared__ int ok;
  uint8_t* me = ws_of(peers, rank);
  if (threadIdx.x == 0) ok = ep_wait_flags(me, EP_FLAGS_COUNTS, G, epoch) &&
                             ep_wait_flags(me, EP_FLAGS_X, G, epoch);
  __syncthreads();
  if (!ok) return;
  const int64_t* c = ep_counts(me, epoch);
  for (int i = threadIdx.x; i < G * EP_MAX_E; i += blockDim.x) cnt[i] = c[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int e = 0; e < E; ++e) {
      lo[e] = acc;
      if (e * G / E == rank)
        for (int s = 0; s < G; ++s) acc += cnt[s * EP_MAX_E + e];
    }
    lo[E] = acc;
    int64_t* out = reinterpret_cast<int64_t*>(me + EP_LOCAL_OFF);
    for (int e = 0; e <= E; ++e) out[e] = lo[e];
  }
  __syncthreads();
  // return address of every received row: (e, s, j) -> source s's y_back
  // row src_off_s[e] + j, where src_off_s is s's own permuted offsets
  uint64_t* rowmap = reinterpret_cast<uint64_t*>(me + EP_ROWMAP);
  for (int e = 0; e < E; ++e) {
    if (e * G / E != rank) continue;
    int64_t base = lo[e];
    for (int s = 0; s < G; ++s) {
      int64_t src_off = 0;
      for (int e2 = 0; e2 < e; ++e2) src_off += cnt[s * EP_MAX_E + e2];
      const int64_t n = cnt[s * EP_MAX_E + e];
      const uint64_t yb = peers[s] + static_cast<uint64_t>(yback_off);
      for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
        rowmap[base + j] = yb + static_cast<uint64_t>(src_off + j) * d * 4;
      base += n;
    }
  }
}

__global__ void ep_wait_back_kernel(uint8_t* ws, int G, unsigned epoch) {
  ep_wait_flags(ws, EP_FLAGS_Y, G, epoch);
}

// ---------------------------------------------------------------- decode (b = 1)
//
// The residual is replicated on every rank; each rank runs the decode kernel
// with its own experts as the resident set (true top-k, identical decisions
// everywhere), so each pick is streamed by exactly its owner.  share: the
// owner stores its picks' fp32 outputs into slot [epoch&1][j] of EVERY
// peer's decode workspace and flags; then every rank combines
// h + sum_j w_j y_j in fixed j order (the single-GPU combine) -> the
// replicated residual of the next layer.
__global__ void ep_decode_share_kernel(const uint64_t* peers, int rank, int G, int k, int d,
                                       const float* y, const uint8_t* is_fast, unsigned epoch) {
  const int s = blockIdx.x / k, j = blockIdx.x - (blockIdx.x / k) * k;
  if (is_fast[j]) {
    float4* dst = reinterpret_cast<float4*>(ws_of(peers, s) + EP_DEC_Y) +
                  (static_cast<int64_t>(epoch & 1) * k + j) * (d / 4);
    const float4* src = reinterpret_cast<const float4*>(y) + static_cast<int64_t>(j) * (d / 4);
    for (int i = threadIdx.x; i < d / 4; i += blockDim.x) dst[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* done = reinterpret_cast<unsigned*>(ws_of(peers, rank) + EP_DONE_SHARE);
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0;
      __threadfence_system();
      for (int q = 0; q < G; ++q)
        st_release_sys(reinterpret_cast<unsigned*>(ws_of(peers, q) + EP_FLAGS_D) + rank, epoch);
    }
  }
}

__global__ void ep_wait_kernel(uint8_t* ws, int64_t flags_off, int G, unsigned epoch) {
  ep_wait_flags(ws, flags_off, G, epoch);
}

// wait for every owner's picks, then out = h + sum_j w_j y_j (fixed j order,
// the combine_dense / fused-decode arithmetic)
__global__ void ep_decode_finish_kernel(uint8_t* ws, int G, int k, int d, const float* h,
                                        const float* w, float* out, unsigned epoch) {
  __shared__ int ok;
  if (threadIdx.x == 0) ok = ep_wait_flags(ws, EP_FLAGS_D, G, epoch);
  __syncthreads();
  const float* y = reinterpret_cast<const float*>(ws + EP_DEC_Y) +
                   static_cast<int64_t>(epoch & 1) * k * d;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
    float o = h[i];
    for (int q = 0; q < k; ++q) o = fmaf(w[q], y[static_cast<int64_t>(q) * d + i], o);
    out[i] = o;
  }
}

}  // namespace daop

using namespace daop;

extern "C" int daop_ep_decode_ws_bytes(int32_t k, int32_t d, int64_t* h_bytes) {
  if (k < 1 || d % 4 != 0) {
    set_error("ep decode: unsupported k=%d d=%d", k, d);
    return DAOP_ERR_UNSUPPORTED;
  }
  *h_bytes = EP_DEC_Y + static_cast<int64_t>(2) * k * d * 4;
  return DAOP_OK;
}

extern "C" int daop_ep_decode_share(const uint64_t* d_peers, int32_t rank, int32_t G, int32_t k,
                                    int32_t d, const float* d_y, const uint8_t* d_is_fast,
                                    uint32_t epoch, daop_stream_t st) {
  if (G < 1 || G > EP_MAX_G || rank < 0 || rank >= G || k < 1 || d % 4 != 0) {
    set_error("ep_decode_share: bad rank/world (%d/%d), k=%d or d=%d", rank, G, k, d);
    return DAOP_ERR_UNSUPPORTED;
  }
  ep_decode_share_kernel<<<G * k, 256, 0, as_stream(st)>>>(d_peers, rank, G, k, d, d_y,
                                                          d_is_fast, epoch);
  DAOP_CHECK_LAUNCH("ep_decode_share");
  return DAOP_OK;
}

extern "C" int daop_ep_decode_wait(void* d_ws, int32_t G, uint32_t epoch, daop_stream_t st) {
  ep_wait_kernel<<<1, 1, 0, as_stream(st)>>>(static_cast<uint8_t*>(d_ws), EP_FLAGS_D, G, epoch);
  DAOP_CHECK_LAUNCH("ep_decode_wait");
  return DAOP_OK;
}

// ---------------------------------------------------------------- C ABI

extern "C" int daop_ep_ws_layout(int32_t G, int32_t E, int32_t d, int64_t cap_recv,
                                 int64_t cap_send, int64_t* total, int64_t* recv_off,
                                 int64_t* yback_off, int64_t* local_off) {
  if (G < 1 || G > EP_MAX_G || E < 1 || E > EP_MAX_E || E % G != 0 || d % 8 != 0 ||
      cap_recv < 0 || cap_send < 0) {
    set_error("ep: unsupported layout (G=%d, E=%d, d=%d): needs G <= %d, E <= %d, E %% G == 0, "
              "d %% 8 == 0", G, E, d, EP_MAX_G, EP_MAX_E);
    return DAOP_ERR_UNSUPPORTED;
  }
  const int64_t r = align_up(EP_ROWMAP + 8 * (cap_recv + 1), 4096);
  const int64_t y = align_up(r + cap_recv * d * 2, 4096);
  *recv_off = r;
  *yback_off = y;
  *local_off = EP_LOCAL_OFF;
  *total = align_up(y + cap_send * d * 4, 4096);
  return DAOP_OK;
}

extern "C" int daop_ep_publish(const uint64_t* d_peers, int32_t rank, int32_t G, int32_t E,
                               const int64_t* d_offsets, uint32_t epoch, daop_stream_t st) {
  if (G < 1 || G > EP_MAX_G || E > EP_MAX_E || rank < 0 || rank >= G) {
    set_error("ep_publish: bad rank/world (%d/%d) or E=%d", rank, G, E);
    return DAOP_ERR_UNSUPPORTED;
  }
  ep_publish_kernel<<<1, 64, 0, as_stream(st)>>>(d_peers, rank, G, E, d_offsets, epoch);
  DAOP_CHECK_LAUNCH("ep_publish");
  return DAOP_OK;
}

extern "C" int daop_ep_dispatch(const uint64_t* d_peers, int32_t rank, int32_t G, int32_t E,
                                int32_t k, int32_t d, const uint16_t* d_x, const int32_t* d_perm,
                                int64_t rows_cap, int64_t recv_off, uint32_t epoch,
                                daop_stream_t st) {
  if (G < 1 || G > EP_MAX_G || E > EP_MAX_E || d % 8 != 0) {
    set_error("ep_dispatch: unsupported shape");
    return DAOP_ERR_UNSUPPORTED;
  }
  int64_t blocks = (rows_cap + EP_WARPS - 1) / EP_WARPS;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  ep_dispatch_kernel<<<static_cast<int>(blocks), EP_WARPS * 32, 0, as_stream(st)>>>(
      d_peers, rank, G, E, k, d, d_x, d_perm, recv_off, epoch);
  DAOP_CHECK_LAUNCH("ep_dispatch");
  return DAOP_OK;
}

extern "C" int daop_ep_recv(const uint64_t* d_peers, int32_t rank, int32_t G, int32_t E,
                            int32_t d, int64_t yback_off, uint32_t epoch, daop_stream_t st) {
  if (G < 1 || G > EP_MAX_G || E > EP_MAX_E) {
    set_error("ep_recv: unsupported shape");
    return DAOP_ERR_UNSUPPORTED;
  }
  ep_recv_kernel<<<1, 512, 0, as_stream(st)>>>(d_peers, rank, G, E, d, yback_off, epoch);
  DAOP_CHECK_LAUNCH("ep_recv");
  return DAOP_OK;
}

extern "C" int daop_ep_wait_back(void* d_ws, int32_t G, uint32_t epoch, daop_stream_t st) {
  ep_wait_back_kernel<<<1, 1, 0, as_stream(st)>>>(static_cast<uint8_t*>(d_ws), G, epoch);
  DAOP_CHECK_LAUNCH("ep_wait_back");
  return DAOP_OK;
}

extern "C" int daop_ep_status(const void* d_ws, int32_t* h_err) {
  unsigned v = 0;
  DAOP_CUDA(cudaMemcpy(&v, static_cast<const uint8_t*>(d_ws) + EP_ERR, 4, cudaMemcpyDeviceToHost));
  *h_err = static_cast<int32_t>(v);
  return DAOP_OK;
}

// ---- CUDA IPC of the workspace (one process per GPU)

static CUresult mem_range(CUdeviceptr* base, size_t* size, CUdeviceptr p) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &q, cudaEnableDefault, &r) ==
            cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Fn>(q);
  }
  if (!fn) return CUDA_ERROR_NOT_SUPPORTED;
  return fn(base, size, p);
}

extern "C" int daop_ep_ipc_handle(const void* d_ptr, void* h_handle, int64_t* h_offset) {
  CUdeviceptr base = 0;
  size_t size = 0;
  if (mem_range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS) {
    set_error("ep_ipc_handle: cuMemGetAddressRange failed");
    return DAOP_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  DAOP_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(h_handle, &h, sizeof(h));
  *h_offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
  return DAOP_OK;
}

extern "C" int daop_ep_ipc_open(const void* h_handle, int64_t offset, void** h_base,
                                void** h_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  void* base = nullptr;
  DAOP_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *h_base = base;
  *h_ptr = static_cast<uint8_t*>(base) + offset;
  return DAOP_OK;
}

extern "C" int daop_ep_ipc_close(void* h_base) {
  DAOP_CUDA(cudaIpcCloseMemHandle(h_base));
  return DAOP_OK;
}

extern "C" int daop_ep_decode_finish(void* d_ws, int32_t G, int32_t k, int32_t d,
                                     const float* d_h, const float* d_w, float* d_out,
                                     uint32_t epoch, daop_stream_t st) {
  ep_decode_finish_kernel<<<(d + 255) / 256, 256, 0, as_stream(st)>>>(
      static_cast<uint8_t*>(d_ws), G, k, d, d_h, d_w, d_out, epoch);
  DAOP_CHECK_LAUNCH("ep_decode_finish");
  return DAOP_OK;
}
