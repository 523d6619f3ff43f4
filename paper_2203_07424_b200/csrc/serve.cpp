// serve.cpp — query splitter / fuser (S1, S2) and the serving runtime (rec_serve).
#include <algorithm>
#include <vector>

#include "model.h"

namespace rec {

// S1: chunks of d, remainder last (reading R14).
struct Chunk {
  int32_t qid, start, len;
  int64_t pos;  // trace row
};

static void split_query(const rec_trace_row& r, int64_t pos, int32_t d, std::vector<Chunk>& out) {
  const int32_t k = (r.size + d - 1) / d;
  for (int32_t c = 0; c < k; ++c)
    out.push_back(Chunk{r.qid, c * d, c < k - 1 ? d : r.size - (k - 1) * d, pos});
}

// S2: number of FIFO-head chunks whose cumulative length stays <= d (at least one).
static int64_t fuse_head(const std::vector<Chunk>& fifo, int64_t head, int32_t d, int64_t* items) {
  int64_t k = 0, tot = 0;
  for (int64_t i = head; i < static_cast<int64_t>(fifo.size()); ++i) {
    if (k > 0 && tot + fifo[i].len > d) break;
    tot += fifo[i].len;
    ++k;
  }
  *items = tot;
  return k;
}

}  // namespace rec

using namespace rec;

extern "C" {

rec_status rec_split_fuse(const rec_trace_row* trace, int64_t n, int32_t max_batch,
                          int32_t* segs_out, int64_t seg_cap, int64_t* batch_start, int64_t bcap,
                          int64_t* nbatches, int64_t* nsegs) {
  if (!trace || !segs_out || !batch_start || !nbatches || !nsegs || n < 0) {
    set_error("null argument");
    return REC_E_INVALID_ARG;
  }
  if (max_batch < 1) {
    set_error("max_batch = %d must be >= 1", max_batch);
    return REC_E_INVALID_ARG;
  }
  std::vector<Chunk> fifo;
  for (int64_t p = 0; p < n; ++p) {
    if (trace[p].size < 1) {
      set_error("trace[%lld].size = %d must be >= 1", (long long)p, trace[p].size);
      return REC_E_INVALID_ARG;
    }
    split_query(trace[p], p, max_batch, fifo);
  }
  if (static_cast<int64_t>(fifo.size()) > seg_cap) {
    set_error("seg_cap = %lld < %zu sub-queries", (long long)seg_cap, fifo.size());
    return REC_E_INVALID_ARG;
  }
  int64_t head = 0, b = 0;
  batch_start[0] = 0;
  while (head < static_cast<int64_t>(fifo.size())) {
    int64_t items = 0;
    const int64_t k = fuse_head(fifo, head, max_batch, &items);
    if (b + 1 > bcap) {
      set_error("bcap = %lld too small", (long long)bcap);
      return REC_E_INVALID_ARG;
    }
    for (int64_t i = head; i < head + k; ++i) {
      segs_out[3 * i] = fifo[i].qid;
      segs_out[3 * i + 1] = fifo[i].start;
      segs_out[3 * i + 2] = fifo[i].len;
    }
    head += k;
    batch_start[++b] = head;
  }
  *nbatches = b;
  *nsegs = head;
  return REC_OK;
}

rec_status rec_serve(rec_model_t m, const rec_trace_row* trace, int64_t n, double sla_ms,
                     const rec_serve_policy* pol, rec_serve_report* out, double* latency_ms,
                     int32_t* batch_log, int64_t log_cap, int64_t* log_rows, float* ctr_out) {
  set_error("rec_serve not built yet");
  return REC_E_UNSUPPORTED;
}

}  // extern "C"
