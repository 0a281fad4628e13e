// DAOP slow tier: SwiGLU expert FFN on the host CPU, weights in pinned host
// memory (the "slow device" of moesim/placement.py:1-8, executed as in
// slow experts of layer l run on the CPU -- on the current
// input below the prediction start layer, on the stale x_{l-1} above it).
//
// Same numeric contract as the GPU experts: bf16 x, bf16 weights, fp32
// accumulation, act = bf16(silu(x.W1) * (x.W3)), y = act . W2 in fp32.
// Inner products use AVX-512 BF16 (vdpbf16ps) when the CPU has it (Sapphire
// Rapids on the GPU box), a scalar loop otherwise.  Rows are split over a
// persistent thread pool.  Compiled as host code inside libdaop_b200.so.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include <immintrin.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <cpuid.h>

#include "common.cuh"

namespace daop {
namespace host {

static inline float bf2f(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f2bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

static float dot_scalar(const uint16_t* a, const uint16_t* b, int n) {
  float acc = 0.f;
  for (int i = 0; i < n; ++i) acc += bf2f(a[i]) * bf2f(b[i]);
  return acc;
}

// two rows against one x in one pass (the W1 and W3 rows of the same unit):
// x is loaded once, four independent accumulator chains, software prefetch
// PF bytes ahead on both weight streams (rows are 8 KB: two 4 KB pages, so the
// hardware streamer alone stalls at every page boundary)
__attribute__((target("avx512f,avx512bf16,avx512bw,avx512vl"))) static void dot2_avx512bf16(
    const uint16_t* x, const uint16_t* a, const uint16_t* b, int n, float* ra, float* rb) {
  constexpr int PF = 2048;  // bytes
  __m512 a0 = _mm512_setzero_ps(), a1 = _mm512_setzero_ps();
  __m512 b0 = _mm512_setzero_ps(), b1 = _mm512_setzero_ps();
  int i = 0;
  for (; i + 64 <= n; i += 64) {
    _mm_prefetch(reinterpret_cast<const char*>(a + i) + PF, _MM_HINT_T0);
    _mm_prefetch(reinterpret_cast<const char*>(a + i) + PF + 64, _MM_HINT_T0);
    _mm_prefetch(reinterpret_cast<const char*>(b + i) + PF, _MM_HINT_T0);
    _mm_prefetch(reinterpret_cast<const char*>(b + i) + PF + 64, _MM_HINT_T0);
    const __m512bh x0 = (__m512bh)_mm512_loadu_si512(x + i);
    const __m512bh x1 = (__m512bh)_mm512_loadu_si512(x + i + 32);
    a0 = _mm512_dpbf16_ps(a0, x0, (__m512bh)_mm512_loadu_si512(a + i));
    a1 = _mm512_dpbf16_ps(a1, x1, (__m512bh)_mm512_loadu_si512(a + i + 32));
    b0 = _mm512_dpbf16_ps(b0, x0, (__m512bh)_mm512_loadu_si512(b + i));
    b1 = _mm512_dpbf16_ps(b1, x1, (__m512bh)_mm512_loadu_si512(b + i + 32));
  }
  float sa = _mm512_reduce_add_ps(_mm512_add_ps(a0, a1));
  float sb = _mm512_reduce_add_ps(_mm512_add_ps(b0, b1));
  for (; i < n; ++i) {
    sa += bf2f(x[i]) * bf2f(a[i]);
    sb += bf2f(x[i]) * bf2f(b[i]);
  }
  *ra = sa;
  *rb = sb;
}

// one long row (W2: ffn elements) with four chains and prefetch
__attribute__((target("avx512f,avx512bf16,avx512bw,avx512vl"))) static float dot_long_avx512bf16(
    const uint16_t* x, const uint16_t* a, int n) {
  constexpr int PF = 2048;
  __m512 c0 = _mm512_setzero_ps(), c1 = _mm512_setzero_ps();
  __m512 c2 = _mm512_setzero_ps(), c3 = _mm512_setzero_ps();
  int i = 0;
  for (; i + 128 <= n; i += 128) {
    const char* pa = reinterpret_cast<const char*>(a + i) + PF;
    _mm_prefetch(pa, _MM_HINT_T0);
    _mm_prefetch(pa + 64, _MM_HINT_T0);
    _mm_prefetch(pa + 128, _MM_HINT_T0);
    _mm_prefetch(pa + 192, _MM_HINT_T0);
    c0 = _mm512_dpbf16_ps(c0, (__m512bh)_mm512_loadu_si512(x + i),
                          (__m512bh)_mm512_loadu_si512(a + i));
    c1 = _mm512_dpbf16_ps(c1, (__m512bh)_mm512_loadu_si512(x + i + 32),
                          (__m512bh)_mm512_loadu_si512(a + i + 32));
    c2 = _mm512_dpbf16_ps(c2, (__m512bh)_mm512_loadu_si512(x + i + 64),
                          (__m512bh)_mm512_loadu_si512(a + i + 64));
    c3 = _mm512_dpbf16_ps(c3, (__m512bh)_mm512_loadu_si512(x + i + 96),
                          (__m512bh)_mm512_loadu_si512(a + i + 96));
  }
  for (; i + 32 <= n; i += 32)
    c0 = _mm512_dpbf16_ps(c0, (__m512bh)_mm512_loadu_si512(x + i),
                          (__m512bh)_mm512_loadu_si512(a + i));
  float r = _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(c0, c1), _mm512_add_ps(c2, c3)));
  for (; i < n; ++i) r += bf2f(x[i]) * bf2f(a[i]);
  return r;
}

static bool have_bf16() {
  static int v = -1;
  if (v < 0) v = __builtin_cpu_supports("avx512bf16") && __builtin_cpu_supports("avx512f") ? 1 : 0;
  return v == 1;
}

static void dot2(const uint16_t* x, const uint16_t* a, const uint16_t* b, int n, float* ra,
                 float* rb) {
  if (have_bf16()) {
    dot2_avx512bf16(x, a, b, n, ra, rb);
  } else {
    *ra = dot_scalar(x, a, n);
    *rb = dot_scalar(x, b, n);
  }
}

static float dot_long(const uint16_t* x, const uint16_t* a, int n) {
  return have_bf16() ? dot_long_avx512bf16(x, a, n) : dot_scalar(x, a, n);
}

// ------------------------------------------------------------------ AMX
// Batched host experts (prefill: tens of tokens per slow expert) are compute
// bound on AVX-512; the 5th-gen Xeon's AMX-BF16 tiles do 16x16x32 per
// TDPBF16PS.  Layout: weights stay row-major (an A tile = 16 weight rows x 32
// k, loaded straight from the pinned pool); the tokens are the B side, packed
// once per call into VNNI pairs ([token block][k block][16 k-pairs][16 tokens]).
// The up pass writes act directly in the down pass's VNNI layout.

struct AmxCfg {
  uint8_t palette;
  uint8_t start_row;
  uint8_t reserved[14];
  uint16_t colsb[16];
  uint8_t rows[16];
};

static bool amx_usable() {
  static int v = -1;
  if (v < 0) {
    unsigned a, b, c, d;
    bool hw = __get_cpuid_count(7, 0, &a, &b, &c, &d) && (d & (1u << 22)) && (d & (1u << 24));
    // Linux: the process must request the tile data state once
    v = hw && syscall(SYS_arch_prctl, 0x1023 /*ARCH_REQ_XCOMP_PERM*/, 18 /*XTILEDATA*/) == 0;
  }
  return v == 1;
}

__attribute__((target("amx-tile,amx-bf16"))) static void amx_config() {
  AmxCfg cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.palette = 1;
  for (int t = 0; t < 8; ++t) {
    cfg.rows[t] = 16;
    cfg.colsb[t] = 64;
  }
  _tile_loadconfig(&cfg);
}

__attribute__((target("amx-tile"))) static void amx_release() { _tile_release(); }

// pack rows [t0, t0+16) of src (n x K bf16, row-major) into VNNI B tiles for
// every k block: dst[kb][r][j] = (src[t0+j][32kb+2r], src[t0+j][32kb+2r+1])
static void pack_vnni(const uint16_t* src, int64_t n, int K, int64_t t0, uint32_t* dst) {
  const int kbs = K / 32;
  for (int kb = 0; kb < kbs; ++kb)
    for (int r = 0; r < 16; ++r)
      for (int j = 0; j < 16; ++j) {
        const int64_t t = t0 + j;
        uint32_t v = 0;
        if (t < n) {
          const uint16_t* p = src + t * K + kb * 32 + 2 * r;
          v = static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 16);
        }
        dst[(static_cast<size_t>(kb) * 16 + r) * 16 + j] = v;
      }
}

// SwiGLU of one AMX output row (16 tokens) in AVX-512: exp(-g) as 2^t with
// a degree-6 polynomial on t - round(t) and the exponent by scalef (~1e-7
// relative, the bf16 act rounding dominates), s = g / (1 + e) * u rounded to
// bf16 like f2bf (nearest-even, NaN kept quiet); the 16 results are written
// to the act pack's VNNI slots (every other 16-bit element, parity `par`) of
// tokens [0, nvalid).  (Replaces a scalar std::exp loop: ~5-10 % of an AMX
// expert at prefill batch sizes, profiles/r02/host_amx_vec_epilogue.txt.)
__attribute__((target("avx512f,avx512bw"))) static inline void swiglu16_vnni(
    const float* g, const float* u, uint16_t* dst, int par, int nvalid) {
  const __m512 gv = _mm512_loadu_ps(g), uv = _mm512_loadu_ps(u);
  __m512 t = _mm512_mul_ps(gv, _mm512_set1_ps(-1.4426950408889634f));
  t = _mm512_min_ps(_mm512_max_ps(t, _mm512_set1_ps(-126.0f)), _mm512_set1_ps(126.0f));
  const __m512 nr = _mm512_roundscale_ps(t, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  const __m512 f = _mm512_sub_ps(t, nr);
  __m512 pl = _mm512_set1_ps(1.535336188319500e-4f);
  pl = _mm512_fmadd_ps(pl, f, _mm512_set1_ps(1.339887440266574e-3f));
  pl = _mm512_fmadd_ps(pl, f, _mm512_set1_ps(9.618437357674640e-3f));
  pl = _mm512_fmadd_ps(pl, f, _mm512_set1_ps(5.550332471162809e-2f));
  pl = _mm512_fmadd_ps(pl, f, _mm512_set1_ps(2.402264791363012e-1f));
  pl = _mm512_fmadd_ps(pl, f, _mm512_set1_ps(6.931472028550421e-1f));
  pl = _mm512_fmadd_ps(pl, f, _mm512_set1_ps(1.0f));
  const __m512 e = _mm512_scalef_ps(pl, nr);
  const __m512 v = _mm512_mul_ps(_mm512_div_ps(gv, _mm512_add_ps(_mm512_set1_ps(1.0f), e)), uv);
  // f2bf: round to nearest even; NaN -> quiet NaN with the same top bits
  const __m512i b = _mm512_castps_si512(v);
  const __m512i rnd = _mm512_add_epi32(
      _mm512_set1_epi32(0x7fff), _mm512_and_si512(_mm512_srli_epi32(b, 16), _mm512_set1_epi32(1)));
  __m512i r = _mm512_srli_epi32(_mm512_add_epi32(b, rnd), 16);
  const __mmask16 nan = _mm512_cmpgt_epu32_mask(_mm512_and_si512(b, _mm512_set1_epi32(0x7fffffff)),
                                                _mm512_set1_epi32(0x7f800000));
  r = _mm512_mask_mov_epi32(r, nan,
                            _mm512_or_si512(_mm512_srli_epi32(b, 16), _mm512_set1_epi32(0x40)));
  if (par) r = _mm512_slli_epi32(r, 16);
  const uint32_t tok = nvalid >= 16 ? 0xffffu : ((1u << nvalid) - 1u);
  uint32_t m = 0;  // 16-bit lane 2j + par for each valid token j
  for (int j = 0; j < 16; ++j)
    if (tok >> j & 1u) m |= 1u << (2 * j + par);
  _mm512_mask_storeu_epi16(dst, m, r);
}

// up: rows [i0, i0+16) of W1/W3 against every token block; act written into
// the down pass's VNNI pack (ffn/32 k-blocks per token block)
__attribute__((target("amx-tile,amx-bf16"))) static void amx_up_block(
    const uint16_t* w1, const uint16_t* w3, int d, int ffn, int64_t i0, const uint32_t* xp,
    int ntb, uint32_t* actp, int64_t n) {
  alignas(64) float g[2][16][16], u[2][16][16];
  const int kbs = d / 32;
  const size_t xtb = static_cast<size_t>(kbs) * 256;           // uint32 per token block
  const size_t atb = static_cast<size_t>(ffn / 32) * 256;
  for (int tb = 0; tb < ntb; tb += 2) {
    const int nb = ntb - tb >= 2 ? 2 : 1;
    _tile_zero(4);
    _tile_zero(5);
    _tile_zero(6);
    _tile_zero(7);
    for (int kb = 0; kb < kbs; ++kb) {
      _tile_loadd(0, w1 + i0 * d + kb * 32, d * 2);
      _tile_loadd(1, w3 + i0 * d + kb * 32, d * 2);
      _tile_loadd(2, xp + tb * xtb + static_cast<size_t>(kb) * 256, 64);
      _tile_dpbf16ps(4, 0, 2);
      _tile_dpbf16ps(5, 1, 2);
      if (nb == 2) {
        _tile_loadd(3, xp + (tb + 1) * xtb + static_cast<size_t>(kb) * 256, 64);
        _tile_dpbf16ps(6, 0, 3);
        _tile_dpbf16ps(7, 1, 3);
      }
    }
    _tile_stored(4, g[0], 64);
    _tile_stored(5, u[0], 64);
    _tile_stored(6, g[1], 64);
    _tile_stored(7, u[1], 64);
    for (int b = 0; b < nb; ++b) {
      uint16_t* ap = reinterpret_cast<uint16_t*>(actp + (tb + b) * atb);
      const int64_t nv = n - static_cast<int64_t>(tb + b) * 16;
      for (int ii = 0; ii < 16; ++ii) {
        const int64_t i = i0 + ii;
        const int64_t kb = i / 32, r = (i % 32) / 2, par = i % 2;
        swiglu16_vnni(g[b][ii], u[b][ii], ap + (kb * 16 + r) * 16 * 2, static_cast<int>(par),
                      static_cast<int>(nv < 16 ? nv : 16));
      }
    }
  }
}

// down: rows [j0, j0+16) of W2 against up to 4 token blocks per pass
__attribute__((target("amx-tile,amx-bf16"))) static void amx_down_block(
    const uint16_t* w2, int d, int ffn, int64_t j0, const uint32_t* actp, int ntb, float* y,
    int64_t n) {
  alignas(64) float c[4][16][16];
  const int kbs = ffn / 32;
  const size_t atb = static_cast<size_t>(kbs) * 256;
  for (int tb = 0; tb < ntb; tb += 4) {
    const int nb = ntb - tb >= 4 ? 4 : ntb - tb;
    _tile_zero(4);
    _tile_zero(5);
    _tile_zero(6);
    _tile_zero(7);
    for (int kb = 0; kb < kbs; ++kb) {
      _tile_loadd(0, w2 + j0 * ffn + kb * 32, ffn * 2);
      _tile_loadd(1, actp + (tb + 0) * atb + static_cast<size_t>(kb) * 256, 64);
      _tile_dpbf16ps(4, 0, 1);
      if (nb > 1) {
        _tile_loadd(2, actp + (tb + 1) * atb + static_cast<size_t>(kb) * 256, 64);
        _tile_dpbf16ps(5, 0, 2);
      }
      if (nb > 2) {
        _tile_loadd(3, actp + (tb + 2) * atb + static_cast<size_t>(kb) * 256, 64);
        _tile_dpbf16ps(6, 0, 3);
      }
      if (nb > 3) {
        _tile_loadd(1, actp + (tb + 3) * atb + static_cast<size_t>(kb) * 256, 64);
        _tile_dpbf16ps(7, 0, 1);
      }
    }
    _tile_stored(4, c[0], 64);
    _tile_stored(5, c[1], 64);
    _tile_stored(6, c[2], 64);
    _tile_stored(7, c[3], 64);
    for (int b = 0; b < nb; ++b)
      for (int jj = 0; jj < 16; ++jj)
        for (int t = 0; t < 16; ++t) {
          const int64_t tok = (tb + b) * 16 + t;
          if (tok < n) y[tok * d + j0 + jj] = c[b][jj][t];
        }
  }
}

// ------------------------------------------------------------------ pool

class Pool {
 public:
  explicit Pool(int n) : n_(n) {
    for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  // run fn(worker, begin, end) over [0, total): split in n_ contiguous parts
  // (grain 0), or in `grain`-sized chunks claimed from a shared counter, so a
  // worker the OS delays (the caller's thread, driver threads share the
  // cores) costs one chunk rather than a whole 1/n_ share
  void run(int64_t total, const std::function<void(int, int64_t, int64_t)>& fn,
           int64_t grain = 0) {
    std::unique_lock<std::mutex> lk(run_m_);
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      total_ = total;
      grain_ = grain;
      next_.store(0, std::memory_order_relaxed);
      pending_ = n_;
      ++gen_;
    }
    cv_.notify_all();
    std::unique_lock<std::mutex> g(m_);
    done_cv_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void loop(int id) {
    uint64_t seen = 0;
    while (true) {
      const std::function<void(int, int64_t, int64_t)>* fn;
      int64_t total, grain;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = fn_;
        total = total_;
        grain = grain_;
      }
      if (grain > 0) {
        for (int64_t a; (a = next_.fetch_add(grain, std::memory_order_relaxed)) < total;)
          (*fn)(id, a, std::min(a + grain, total));
      } else {
        const int64_t a = total * id / n_, b = total * (id + 1) / n_;
        if (a < b) (*fn)(id, a, b);
      }
      {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_cv_.notify_all();
      }
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_, run_m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int, int64_t, int64_t)>* fn_ = nullptr;
  int64_t total_ = 0, grain_ = 0;
  std::atomic<int64_t> next_{0};
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// one pool per thread count, created on first use and never destroyed: a
// caller asking for another size can never free a pool another thread is
// running on (pools are few -- one per distinct `threads` value)
static Pool* pool_for(int threads) {
  static std::mutex m;
  static std::map<int, Pool*>* pools = new std::map<int, Pool*>();
  std::lock_guard<std::mutex> g(m);
  Pool*& p = (*pools)[threads];
  if (!p) p = new Pool(threads);
  return p;
}

}  // namespace host
}  // namespace daop

using namespace daop;

// chunk sizes of the GEMV phases (rows; 0 = static split): ~0.5-1 MB of
// weights per claim.  Settable for sweeps (daop_host_set_grain).
static int64_t g_grain_up = 32, g_grain_down = 16;

extern "C" int daop_host_set_grain(int64_t up, int64_t down) {
  g_grain_up = up < 0 ? 0 : up;
  g_grain_down = down < 0 ? 0 : down;
  return DAOP_OK;
}

extern "C" int daop_host_expert_ffn(const uint16_t* x, int64_t n, const uint16_t* w1,
                                    const uint16_t* w3, const uint16_t* w2, int32_t d,
                                    int32_t ffn, float* y, uint16_t* act_scratch,
                                    int32_t threads) {
  if (n < 0 || d <= 0 || ffn <= 0) {
    set_error("host_expert_ffn: invalid shape");
    return DAOP_ERR_SHAPE;
  }
  if (n == 0) return DAOP_OK;
  // default: one worker per hardware thread, rows claimed in chunks
  // (scripts/host_threads_probe.py, 16 cores, 8x7B expert: 1.90 ms = 185 GB/s,
  // vs 2.2-2.9 ms with static shares, where one delayed worker stalls all)
  if (threads < 1) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  host::Pool* pool = host::pool_for(threads);
  if (n >= 16 && d % 32 == 0 && ffn % 32 == 0 && host::amx_usable()) {
    // batched experts on AMX tiles (prefill slow tier)
    const int ntb = static_cast<int>((n + 15) / 16);
    std::vector<uint32_t> xp(static_cast<size_t>(ntb) * (d / 32) * 256);
    std::vector<uint32_t> actp(static_cast<size_t>(ntb) * (ffn / 32) * 256, 0u);
    pool->run(ntb, [&](int, int64_t a, int64_t b) {
      for (int64_t tb = a; tb < b; ++tb)
        host::pack_vnni(x, n, d, tb * 16, xp.data() + tb * (d / 32) * 256);
    });
    pool->run(ffn / 16, [&](int, int64_t a, int64_t b) {
      if (a >= b) return;
      host::amx_config();
      for (int64_t blk = a; blk < b; ++blk)
        host::amx_up_block(w1, w3, d, ffn, blk * 16, xp.data(), ntb, actp.data(), n);
      host::amx_release();
    }, g_grain_up > 0 ? 4 : 0);
    pool->run(d / 16, [&](int, int64_t a, int64_t b) {
      if (a >= b) return;
      host::amx_config();
      for (int64_t blk = a; blk < b; ++blk)
        host::amx_down_block(w2, d, ffn, blk * 16, actp.data(), ntb, y, n);
      host::amx_release();
    }, g_grain_down > 0 ? 2 : 0);
    if (act_scratch) {  // unpack act for callers that asked for it
      for (int64_t t = 0; t < n; ++t)
        for (int i = 0; i < ffn; ++i) {
          const int64_t tb = t / 16, j = t % 16, kb = i / 32, r = (i % 32) / 2, par = i % 2;
          act_scratch[t * ffn + i] = reinterpret_cast<const uint16_t*>(
              actp.data() + tb * (ffn / 32) * 256)[((kb * 16 + r) * 16 + j) * 2 + par];
        }
    }
    return DAOP_OK;
  }
  std::vector<uint16_t> own;
  uint16_t* act = act_scratch;
  if (!act) {
    own.resize(static_cast<size_t>(n) * ffn);
    act = own.data();
  }
  // up: rows i of W1/W3 split over workers; every token reuses the row from cache
  pool->run(ffn, [&](int, int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      const uint16_t* r1 = w1 + i * d;
      const uint16_t* r3 = w3 + i * d;
      for (int64_t t = 0; t < n; ++t) {
        float g, u;
        host::dot2(x + t * d, r1, r3, d, &g, &u);
        const float s = g / (1.0f + std::exp(-g));
        act[t * ffn + i] = host::f2bf(s * u);
      }
    }
  }, g_grain_up);
  // down: rows j of W2
  pool->run(d, [&](int, int64_t a, int64_t b) {
    for (int64_t j = a; j < b; ++j) {
      const uint16_t* r2 = w2 + j * ffn;
      for (int64_t t = 0; t < n; ++t) y[t * d + j] = host::dot_long(act + t * ffn, r2, ffn);
    }
  }, g_grain_down);
  return DAOP_OK;
}

// The expert restricted to ffn rows [r0, r1): act rows r0..r1-1 and
// y = W2[:, r0:r1] . act[r0:r1] -- the host's share of a slow expert whose
// rows [0, r0) the GPU computes from a copy pulled over PCIe (the host's
// DRAM serves both: ~200 GB/s together vs ~170 for the host alone).
// Decode-sized n (< 16, the AVX-512 path); y (n, d) fp32 is overwritten.
extern "C" int daop_host_expert_ffn_rows(const uint16_t* x, int64_t n, const uint16_t* w1,
                                         const uint16_t* w3, const uint16_t* w2, int32_t d,
                                         int32_t ffn, int32_t r0, int32_t r1, float* y,
                                         int32_t threads) {
  if (n < 0 || n >= 16 || d <= 0 || ffn <= 0 || r0 < 0 || r1 > ffn || r0 >= r1) {
    set_error("host_expert_ffn_rows: invalid shape (n=%lld d=%d ffn=%d rows %d..%d); n < 16",
              static_cast<long long>(n), d, ffn, r0, r1);
    return DAOP_ERR_SHAPE;
  }
  if (n == 0) return DAOP_OK;
  if (threads < 1) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  host::Pool* pool = host::pool_for(threads);
  const int nr = r1 - r0;
  std::vector<uint16_t> act(static_cast<size_t>(n) * nr);
  pool->run(nr, [&](int, int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      const uint16_t* q1 = w1 + (r0 + i) * d;
      const uint16_t* q3 = w3 + (r0 + i) * d;
      for (int64_t t = 0; t < n; ++t) {
        float g, u;
        host::dot2(x + t * d, q1, q3, d, &g, &u);
        const float sv = g / (1.0f + std::exp(-g));
        act[t * nr + i] = host::f2bf(sv * u);
      }
    }
  }, g_grain_up);
  pool->run(d, [&](int, int64_t a, int64_t b) {
    for (int64_t j = a; j < b; ++j) {
      const uint16_t* q2 = w2 + j * ffn + r0;
      for (int64_t t = 0; t < n; ++t) y[t * d + j] = host::dot_long(act.data() + t * nr, q2, nr);
    }
  }, g_grain_down);
  return DAOP_OK;
}

// profiling aid: read `bytes` of host memory with the host tier's thread pool
// (64 B vector loads, contiguous split) -- the bandwidth ceiling of the slow
// tier's GEMV, measured on the same threads
__attribute__((target("avx512f"))) static double sum_range(const uint8_t* p, int64_t n) {
  __m512i acc = _mm512_setzero_si512();
  int64_t i = 0;
  for (; i + 256 <= n; i += 256) {
    acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i));
    acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i + 64));
    acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i + 128));
    acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i + 192));
  }
  return static_cast<double>(_mm512_reduce_add_epi64(acc) & 0xffff);
}

extern "C" int daop_host_stream_read(const void* p, int64_t bytes, int32_t threads,
                                     double* checksum) {
  if (threads < 1) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  host::Pool* pool = host::pool_for(threads);
  std::vector<double> part(threads, 0.0);
  const int64_t lines = bytes / 256;
  pool->run(lines, [&](int id, int64_t a, int64_t b) {
    part[id] = sum_range(static_cast<const uint8_t*>(p) + a * 256, (b - a) * 256);
  });
  double c = 0.0;
  for (double v : part) c += v;
  *checksum = c;
  return DAOP_OK;
}

extern "C" int daop_host_caps(int32_t* avx512_bf16, int32_t* hw_threads) {
  *avx512_bf16 = (host::have_bf16() ? 1 : 0) | (host::amx_usable() ? 2 : 0);
  *hw_threads = static_cast<int32_t>(std::thread::hardware_concurrency());
  return DAOP_OK;
}

// Pinned host pool for the slow tier / migration source (HostExpertPool):
// anonymous mmap with transparent huge pages, first-touched by every core in
// parallel, then registered with the driver (cudaHostRegister).  Measured on
// the GPU box (scripts/pin_probe.py, 16 GB): 1.8 s against 9.2 s for
// cudaHostAlloc (torch pin_memory), whose 4 KB pages are faulted by one
// thread -- 90 GB of Mixtral-8x7B experts in ~10 s instead of ~60 s.
extern "C" int daop_host_pool_alloc(int64_t bytes, int32_t threads, void** out,
                                    int32_t* registered) {
  *out = nullptr;
  *registered = 0;
  if (bytes <= 0) {
    set_error("host_pool_alloc: bytes must be positive");
    return DAOP_ERR_SHAPE;
  }
  void* p = mmap(nullptr, static_cast<size_t>(bytes), PROT_READ | PROT_WRITE,
                 MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) {
    set_error("host_pool_alloc: mmap of %lld bytes failed", static_cast<long long>(bytes));
    return DAOP_ERR_CUDA;
  }
  madvise(p, static_cast<size_t>(bytes), MADV_HUGEPAGE);
  if (threads < 1) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  host::Pool* pool = host::pool_for(threads);
  const int64_t chunk = int64_t(64) << 20;  // 64 MB first-touch claims
  pool->run((bytes + chunk - 1) / chunk, [&](int, int64_t a, int64_t b) {
    for (int64_t c = a; c < b; ++c) {
      const int64_t off = c * chunk;
      std::memset(static_cast<uint8_t*>(p) + off, 0, static_cast<size_t>(std::min(chunk, bytes - off)));
    }
  }, 1);
  const cudaError_t e = cudaHostRegister(p, static_cast<size_t>(bytes), cudaHostRegisterPortable);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    // no GPU (the build container): host-tier memory only, nothing to pin for
    cudaGetLastError();
    *out = p;
    return DAOP_OK;
  }
  if (e != cudaSuccess) {
    munmap(p, static_cast<size_t>(bytes));
    set_error("host_pool_alloc: cudaHostRegister: %s", cudaGetErrorString(e));
    return DAOP_ERR_CUDA;
  }
  *registered = 1;
  *out = p;
  return DAOP_OK;
}

extern "C" int daop_host_pool_free(void* p, int64_t bytes, int32_t registered) {
  if (!p) return DAOP_OK;
  if (registered) cudaHostUnregister(p);
  munmap(p, static_cast<size_t>(bytes));
  return DAOP_OK;
}
