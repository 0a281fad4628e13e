// Native writer for the moesim JSON-Lines trace format.
//
// Follows moesim/trace.py:328-362 (save_trace / _fmt_vector): every score is
// printed with "%.17g" (Python's format(float(v), ".17g") -- both are
// correctly rounded, same exponent and trailing-zero rules), token records
// are '{"phase":"...","token_index":t,"layers":[{"true_scores":[...],
// "predicted_scores":[...]|null},...]}' one per line.  The header line is
// written by the Python side (json.dumps(sort_keys=True)).  Tokens are
// formatted in parallel chunks on host threads and concatenated in order, so
// the bytes are identical to the reference writer's for any thread count.
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace daop {
namespace {

void append_vector(std::string& o, const double* v, int E) {
  char buf[40];
  o.push_back('[');
  for (int e = 0; e < E; ++e) {
    if (e) o.push_back(',');
    const int n = std::snprintf(buf, sizeof(buf), "%.17g", v[e]);
    o.append(buf, n);
  }
  o.push_back(']');
}

void format_tokens(const double* tr, const double* pr, const uint8_t* mask, int64_t t0,
                   int64_t t1, int L, int E, const char* phase, std::string& o) {
  char head[96];
  for (int64_t t = t0; t < t1; ++t) {
    const int n = std::snprintf(head, sizeof(head), "{\"phase\":\"%s\",\"token_index\":%lld,\"layers\":[",
                                phase, static_cast<long long>(t));
    o.append(head, n);
    for (int l = 0; l < L; ++l) {
      if (l) o.push_back(',');
      const int64_t off = (t * L + l) * static_cast<int64_t>(E);
      o.append("{\"true_scores\":");
      append_vector(o, tr + off, E);
      o.append(",\"predicted_scores\":");
      if (mask[t * L + l]) append_vector(o, pr + off, E);
      else o.append("null");
      o.push_back('}');
    }
    o.append("]}\n");
  }
}

}  // namespace
}  // namespace daop

using namespace daop;

extern "C" int daop_trace_format_phase(const double* true_scores, const double* pred_scores,
                                       const uint8_t* mask, int64_t T, int32_t L, int32_t E,
                                       int32_t phase, char* out, int64_t cap, int64_t* written) {
  if (T < 0 || L < 1 || E < 2 || (phase != 0 && phase != 1) || !written) {
    set_error("trace_format_phase: bad arguments (T=%lld L=%d E=%d phase=%d)",
              static_cast<long long>(T), L, E, phase);
    return DAOP_ERR_SHAPE;
  }
  const char* name = phase == 0 ? "prefill" : "decode";
  unsigned nt = std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  const int64_t work = T * L * E;
  if (work < (1 << 16)) nt = 1;
  if (static_cast<int64_t>(nt) > T) nt = T > 0 ? static_cast<unsigned>(T) : 1;
  std::vector<std::string> parts(nt);
  std::vector<std::thread> th;
  const int64_t per = (T + nt - 1) / nt;
  for (unsigned i = 0; i < nt; ++i) {
    const int64_t t0 = i * per, t1 = T < (i + 1) * per ? T : (i + 1) * per;
    if (t0 >= t1) continue;
    auto job = [&, t0, t1, i]() {
      parts[i].reserve(static_cast<size_t>((t1 - t0) * L * (48 + 2 * 24 * E)));
      format_tokens(true_scores, pred_scores, mask, t0, t1, L, E, name, parts[i]);
    };
    if (nt == 1) job();
    else th.emplace_back(job);
  }
  for (auto& x : th) x.join();
  int64_t total = 0;
  for (auto& p : parts) total += static_cast<int64_t>(p.size());
  *written = total;
  if (!out) return DAOP_OK;  // size query
  if (total > cap) {
    set_error("trace_format_phase: %lld bytes do not fit the %lld-byte buffer",
              static_cast<long long>(total), static_cast<long long>(cap));
    return DAOP_ERR_SHAPE;
  }
  for (auto& p : parts) {
    std::memcpy(out, p.data(), p.size());
    out += p.size();
  }
  return DAOP_OK;
}
