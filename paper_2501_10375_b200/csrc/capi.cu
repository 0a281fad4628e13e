// Library plumbing + host decision entry points (placement.py / policies.py).
//
// The host decisions are pure C++ restatements of the reference, bit-exact:
// they are pinned by tests/test_host_decisions.py against the golden vectors
// recorded from moesim itself.
#include <cstdlib>
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <numeric>
#include <thread>
#include <vector>

#include "common.cuh"
#include "decide.cuh"
#include "rng.cuh"

namespace daop {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %d (%s) at %s", static_cast<int>(e), cudaGetErrorString(e), what);
  return DAOP_ERR_CUDA;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("DAOP_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

}  // namespace daop

using namespace daop;

extern "C" {

const char* daop_last_error(void) { return g_err; }

int daop_version(void) { return 1; }

int daop_device_info(int* sms, int* major, int* minor) {
  int dev = 0;
  DAOP_CUDA(cudaGetDevice(&dev));
  DAOP_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  DAOP_CUDA(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev));
  DAOP_CUDA(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev));
  return DAOP_OK;
}

// One synchronous host step of a captured graph: stage the caller's host
// input into the graph's pinned source buffer, launch, wait.  The end-to-end
// decode call (engine.decode_host) runs entirely here, with no Python between
// the staging copy, the launch and the synchronisation.
static int g_graph_step_spin = 0;
int daop_graph_step_mode(int32_t spin) {
  g_graph_step_spin = spin;
  return DAOP_OK;
}

int daop_graph_step(void* graph_exec, daop_stream_t stream, const void* h_src, void* h_staging,
                    int64_t bytes) {
  if (!graph_exec) {
    set_error("graph_step: null graph");
    return DAOP_ERR_UNSUPPORTED;
  }
  if (bytes > 0 && h_src && h_src != h_staging) memcpy(h_staging, h_src, static_cast<size_t>(bytes));
  DAOP_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), as_stream(stream)));
  if (g_graph_step_spin) {
    // busy-poll: no sleep / yield between the kernel's last store and the return
    cudaError_t e;
    while ((e = cudaStreamQuery(as_stream(stream))) == cudaErrorNotReady) {
    }
    DAOP_CUDA(e);
  } else {
    DAOP_CUDA(cudaStreamSynchronize(as_stream(stream)));
  }
  return DAOP_OK;
}

// placement.py:123-125 -- math.floor(ecr * L * E), left to right in double
// The GPU's share of a slow expert: rows [0, rows) of W1 and W3 and columns
// [0, rows) of W2, pulled from the expert's pinned host copy over PCIe into a
// staging slot laid out as an expert with ffn = rows ([W1 | W3 | W2 (d x
// rows)]), on `stream` (three async copies; W2's columns as one 2-D copy).
int daop_slow_split_pull(const uint16_t* h_w1, const uint16_t* h_w3, const uint16_t* h_w2,
                         int32_t d, int32_t ffn, int32_t rows, uint16_t* d_stage,
                         daop_stream_t stream) {
  if (d <= 0 || ffn <= 0 || rows <= 0 || rows > ffn) {
    set_error("slow_split_pull: invalid shape (d=%d ffn=%d rows=%d)", d, ffn, rows);
    return DAOP_ERR_SHAPE;
  }
  cudaStream_t st = as_stream(stream);
  const size_t rb = static_cast<size_t>(rows) * d * 2;
  DAOP_CUDA(cudaMemcpyAsync(d_stage, h_w1, rb, cudaMemcpyHostToDevice, st));
  DAOP_CUDA(cudaMemcpyAsync(d_stage + static_cast<size_t>(rows) * d, h_w3, rb,
                            cudaMemcpyHostToDevice, st));
  DAOP_CUDA(cudaMemcpy2DAsync(d_stage + 2 * static_cast<size_t>(rows) * d,
                              static_cast<size_t>(rows) * 2, h_w2, static_cast<size_t>(ffn) * 2,
                              static_cast<size_t>(rows) * 2, static_cast<size_t>(d),
                              cudaMemcpyHostToDevice, st));
  return DAOP_OK;
}

int daop_slot_budget(double ecr, int32_t L, int32_t E, int64_t* budget) {
  double v = (ecr * static_cast<double>(L)) * static_cast<double>(E);
  if (!std::isfinite(v)) {
    set_error("slot budget of ecr=%g is not finite", ecr);
    return DAOP_ERR_BUDGET;
  }
  *budget = static_cast<int64_t>(std::floor(v));
  return DAOP_OK;
}

// placement.py:128-185
int daop_placement_init(const double* calib, int32_t L, int32_t E, double ecr, uint8_t* on_fast,
                        int64_t* budget_out) {
  if (L < 1 || E < 2) {
    set_error("invalid calibration shape (%d, %d)", L, E);
    return DAOP_ERR_SHAPE;
  }
  if (!(0.0 < ecr && ecr <= 1.0)) {  // :151-152 (NaN fails too)
    set_error("ecr must be in (0, 1], got %g", ecr);
    return DAOP_ERR_BUDGET;
  }
  int64_t budget = 0;
  int rc = daop_slot_budget(ecr, L, E, &budget);
  if (rc) return rc;
  if (budget < L) {  // :154-157
    set_error("budget %lld cannot give every one of %d layers a slot",
              static_cast<long long>(budget), L);
    return DAOP_ERR_BUDGET;
  }
  const int64_t base = budget / L, rem = budget - base * L;
  std::fill(on_fast, on_fast + static_cast<size_t>(L) * E, uint8_t(0));
  std::vector<int> order(E);
  for (int l = 0; l < L; ++l) {  // :166-169 per-layer top-base by (-v, j)
    const double* v = calib + static_cast<size_t>(l) * E;
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return -v[a] < -v[b]; });
    for (int64_t i = 0; i < base && i < E; ++i) on_fast[static_cast<size_t>(l) * E + order[i]] = 1;
  }
  if (rem) {  // :171-183 remainder by (-v, l, j), at most one extra per layer
    std::vector<std::pair<int, int>> cand;
    for (int l = 0; l < L; ++l)
      for (int j = 0; j < E; ++j)
        if (!on_fast[static_cast<size_t>(l) * E + j]) cand.emplace_back(l, j);
    std::stable_sort(cand.begin(), cand.end(), [&](const auto& a, const auto& b) {
      return -calib[static_cast<size_t>(a.first) * E + a.second] <
             -calib[static_cast<size_t>(b.first) * E + b.second];
    });  // candidates were generated in (l, j) order, so stability breaks ties
    std::vector<uint8_t> granted(L, 0);
    int64_t n_granted = 0;
    for (const auto& c : cand) {
      if (n_granted == rem) break;
      if (granted[c.first]) continue;
      on_fast[static_cast<size_t>(c.first) * E + c.second] = 1;
      granted[c.first] = 1;
      ++n_granted;
    }
  }
  *budget_out = budget;
  return DAOP_OK;
}

// placement.py:188-237 (Alg. 1), exact rational threshold num/den
int daop_allocate(const uint8_t* on_fast, const int64_t* counts, int32_t L, int32_t E,
                  int64_t thr_num, int64_t thr_den, uint8_t* out, int64_t* events,
                  int32_t* n_events) {
  if (thr_den <= 0) {
    set_error("threshold denominator must be positive");
    return DAOP_ERR_CONFIG;
  }
  for (int64_t i = 0; i < static_cast<int64_t>(L) * E; ++i) {
    if (counts[i] < 0) {
      set_error("prefill counts must be nonnegative integers");
      return DAOP_ERR_SHAPE;
    }
  }
  const int swap_num = E / 2;  // :213
  int ne = 0;
  std::vector<int> hot, cold;
  for (int l = 0; l < L; ++l) {
    const uint8_t* in = on_fast + static_cast<size_t>(l) * E;
    uint8_t* o = out + static_cast<size_t>(l) * E;
    const int64_t* act = counts + static_cast<size_t>(l) * E;
    std::copy(in, in + E, o);
    hot.clear();
    cold.clear();
    for (int j = 0; j < E; ++j) (in[j] ? cold : hot).push_back(j);
    // :221 hot = slow sorted by (-act, j); :222 cold = cached sorted by (act, j)
    std::stable_sort(hot.begin(), hot.end(), [&](int a, int b) { return act[a] > act[b]; });
    std::stable_sort(cold.begin(), cold.end(), [&](int a, int b) { return act[a] < act[b]; });
    const int pairs = std::min<int>(swap_num, std::min(hot.size(), cold.size()));
    for (int i = 0; i < pairs; ++i) {
      const int h = hot[i], c = cold[i];
      // :224 Fraction(h) >= Fraction(num, den) * c  <=>  h*den >= num*c
      const __int128 lhs = static_cast<__int128>(act[h]) * thr_den;
      const __int128 rhs = static_cast<__int128>(thr_num) * act[c];
      if (lhs >= rhs) {
        o[c] = 0;
        o[h] = 1;
        int64_t* ev = events + static_cast<size_t>(ne) * 5;
        ev[0] = l;
        ev[1] = h;
        ev[2] = c;
        ev[3] = act[h];
        ev[4] = act[c];
        ++ne;
      }
    }
  }
  *n_events = ne;
  return DAOP_OK;
}

int daop_degrade_f64(const double* scores, int32_t E, int32_t* sel, int32_t k,
                     const uint8_t* fast, int32_t* drop, int32_t* sub, int32_t* n_deg) {
  for (int q = 0; q < k; ++q) {
    if (sel[q] < 0 || sel[q] >= E) {
      set_error("selection id %d out of range", sel[q]);
      return DAOP_ERR_SHAPE;
    }
  }
  *n_deg = degrade(scores, E, sel, k, fast, drop, sub);
  return DAOP_OK;
}

int daop_plan_token_f64(const double* tr, const double* pr, const uint8_t* pmask,
                        const uint8_t* on_fast, int32_t L, int32_t E, int32_t k, int32_t start,
                        int32_t engine, int32_t graceful, int32_t* sel, uint8_t* is_fast,
                        int32_t* drop, int32_t* sub, int32_t* n_deg) {
  if (k < 1 || k > E) {
    set_error("top_k must be in [1, %d], got %d", E, k);
    return DAOP_ERR_SHAPE;
  }
  if (engine != DAOP_ENGINE_DAOP && engine != DAOP_ENGINE_FIDDLER) {
    set_error("engine %d has no native planner", engine);
    return DAOP_ERR_CONFIG;
  }
  const bool daop_engine = engine == DAOP_ENGINE_DAOP;
  for (int l = 0; l < L; ++l) {
    const size_t o = static_cast<size_t>(l) * E, ok = static_cast<size_t>(l) * k;
    const bool present = l > 0 && pmask[l - 1];
    int nd = plan_layer(l, tr + o, l > 0 ? pr + o - E : nullptr, present, on_fast + o, E, k, start,
                        daop_engine, graceful != 0, sel + ok, is_fast + ok, drop + ok, sub + ok);
    if (nd < 0) {
      set_error("layer %d record carries no prediction for layer %d", l - 1, l);
      return DAOP_ERR_PREDICTION_MISSING;
    }
    n_deg[l] = nd;
  }
  return DAOP_OK;
}

// policies.py:120-127 _LayerCache.insert on row lu (E entries, -1 = absent)
static int lru_insert(int64_t* lu, int E, int cap, int e, int64_t step, int* evicted) {
  *evicted = -1;
  if (lu[e] < 0) {
    int members = 0;
    for (int c = 0; c < E; ++c) members += lu[c] >= 0;
    if (members >= cap) {
      int ev = -1;
      for (int c = 0; c < E; ++c)  // min (last_use, id)
        if (lu[c] >= 0 && (ev < 0 || lu[c] < lu[ev])) ev = c;
      if (ev < 0) return -1;  // capacity 0
      lu[ev] = -1;
      *evicted = ev;
    }
  }
  lu[e] = step;
  return 0;
}

int daop_lru_plan_layer(int32_t l, int32_t L, int32_t E, int32_t k, int32_t engine, int32_t start,
                        const double* tr, const double* pr, int64_t* last_use,
                        const int32_t* capacity, int64_t* step, int32_t* sel, int32_t* mig,
                        int32_t* mig_ev, int32_t* n_mig, int32_t* pf, int32_t* pf_ev,
                        int32_t* n_pf) {
  if (k < 1 || k > E || l < 0 || l >= L) {
    set_error("lru_plan_layer: bad shape (layer %d of %d, E=%d, k=%d)", l, L, E, k);
    return DAOP_ERR_SHAPE;
  }
  if (engine != DAOP_ENGINE_ONDEMAND && engine != DAOP_ENGINE_PREFETCH) {
    set_error("engine %d has no LRU planner", engine);
    return DAOP_ERR_CONFIG;
  }
  const int64_t st = ++*step;
  int64_t* lu = last_use + static_cast<size_t>(l) * E;
  int need[64];
  if (k > 64) {
    set_error("lru_plan_layer: k=%d > 64", k);
    return DAOP_ERR_UNSUPPORTED;
  }
  topk_scan(tr, E, k, need);
  for (int q = 0; q < k; ++q) sel[q] = need[q];
  // absent = sorted(need not cached); touch the cached ones (policies.py:181-186)
  int nm = 0;
  for (int e = 0; e < E; ++e)
    for (int q = 0; q < k; ++q)
      if (need[q] == e && lu[e] < 0) mig[nm++] = e;
  for (int q = 0; q < k; ++q)
    if (lu[need[q]] >= 0) lu[need[q]] = st;
  for (int i = 0; i < nm; ++i) {
    if (lru_insert(lu, E, capacity[l], mig[i], st, &mig_ev[i]) < 0) {
      set_error("layer %d cache has no capacity", l);
      return DAOP_ERR_CONFIG;
    }
  }
  *n_mig = nm;
  *n_pf = 0;
  if (engine == DAOP_ENGINE_PREFETCH && l + 1 < L && l + 1 >= start) {  // :223-236
    if (!pr) {
      set_error("layer %d record carries no prediction for layer %d", l, l + 1);
      return DAOP_ERR_PREDICTION_MISSING;
    }
    int ptop[64];
    topk_scan(pr, E, k, ptop);
    int64_t* nlu = last_use + static_cast<size_t>(l + 1) * E;
    int np = 0;
    for (int e = 0; e < E; ++e)
      for (int q = 0; q < k; ++q)
        if (ptop[q] == e && nlu[e] < 0) pf[np++] = e;
    for (int i = 0; i < np; ++i) {
      if (lru_insert(nlu, E, capacity[l + 1], pf[i], st, &pf_ev[i]) < 0) {
        set_error("layer %d cache has no capacity", l + 1);
        return DAOP_ERR_CONFIG;
      }
    }
    *n_pf = np;
  }
  return DAOP_OK;
}

int daop_fill_uniform_bf16_host(uint16_t* dst, int64_t n, uint64_t seed, uint64_t tag, float scale,
                                int64_t off, int32_t threads) {
  const uint64_t key = stream_key(seed, tag);
  if (threads < 1) threads = 1;
  auto work = [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      uint64_t z = mix64(key + (static_cast<uint64_t>(i + off) + 1ull) * kGolden);
      float u = static_cast<float>(static_cast<uint32_t>(z >> 40)) * 1.1920928955078125e-07f - 1.0f;
      float v = u * scale;
      uint32_t bits;
      std::memcpy(&bits, &v, 4);
      bits = (bits + 0x7FFFu + ((bits >> 16) & 1u)) >> 16;
      dst[i] = static_cast<uint16_t>(bits);
    }
  };
  std::vector<std::thread> pool;
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    int64_t a = t * chunk, b = std::min(n, a + chunk);
    if (a < b) pool.emplace_back(work, a, b);
  }
  for (auto& th : pool) th.join();
  return DAOP_OK;
}

}  // extern "C"
