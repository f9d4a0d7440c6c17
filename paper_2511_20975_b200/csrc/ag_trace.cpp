// Trace I/O of accurate-configuration sets: the
// reference's External Interfaces clause -- a
// line-delimited trace of request id, arrival timestamp and the accurate set,
// "bitmap over canonical config enumeration for M^N <= 4096, explicit list
// otherwise".  The reference ships no writer for it (its JSONL run trace,
// src/simulation.cpp:408-461, records per-request outcomes, not sets), so the
// format below is this library's reading of the clause:
//
//   {"id": <RequestId>, "arrival": <seconds, %.17g>,
//    "accurate": {"encoding": "bitmap", "size": M^N, "bits": "<hex>"}}
//     bits: ceil(M^N / 8) bytes, two hex digits each, byte k holding
//     canonical indices 8k .. 8k+7 in bits 0..7 (little-endian bit order)
//   {"id": ..., "arrival": ...,
//    "accurate": {"encoding": "list", "size": M^N, "members": [i0, i1, ...]}}
//     members ascending canonical indices
//
// The sets are enumerated on the device (ag_route_enumerate, oracle router =
// AccurateSet::contains, accuracy.cpp:116-124), the text is formatted here.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ag_internal.h"

using agb::fail;

extern "C" int ag_trace_write(ag_ctx* ctx, const ag_truth* th, const double* arrival, const char* path,
                              uint64_t* bytes_written) {
  agb::DeviceGuard device_guard(ctx ? ctx->device : -1);
  if (!ctx || !th || !path) return fail(AG_ERR_VALIDATION, "null argument");
  const int R = th->n_requests;
  if (R < 0) return fail(AG_ERR_VALIDATION, "negative request count");
  const ag_space* sp = ctx->space;
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N < 2^32 and N <= 32");
  const uint64_t S = sp->size;
  const bool bitmap = S <= 4096;
  FILE* f = std::fopen(path, "w");
  if (!f) return fail(AG_ERR_IO, std::string("cannot open trace file: ") + path);
  const ag_router oracle{AG_ROUTER_ORACLE, 0.0, 0.0, 0, 0.0};
  // requests in chunks bounded to 2^26 enumerated configurations
  const int chunk = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)std::max(R, 1), (1ull << 26) / S));
  std::vector<uint64_t> counts, offsets;
  std::vector<uint32_t> idx;
  std::string line;
  uint64_t written = 0;
  int rc = AG_OK;
  for (int r0 = 0; r0 < R && rc == AG_OK; r0 += chunk) {
    const int n = std::min(chunk, R - r0);
    // the chunk's rows of the CSR truth batch (pointers shifted, offsets kept)
    ag_truth t = *th;
    t.n_requests = n;
    t.request_ids = th->request_ids + r0;
    t.seed_ptr = th->seed_ptr + r0;
    t.removed_ptr = th->removed_ptr + r0;
    counts.assign(n, 0);
    offsets.assign((size_t)n + 1, 0);
    // the chunk's member total first (counts only), then exactly that much
    // host memory for the indices
    uint64_t total = 0;
    rc = ag_route_enumerate_host(ctx, &t, &oracle, 0, S, 0, counts.data(), offsets.data(), nullptr, 0, &total);
    if (rc) break;
    idx.assign((size_t)total + 1, 0);
    rc = ag_route_enumerate_host(ctx, &t, &oracle, 0, S, 0, counts.data(), offsets.data(), idx.data(), idx.size(),
                                 &total);
    if (rc) break;
    for (int i = 0; i < n; ++i) {
      const int r = r0 + i;
      char head[96];
      std::snprintf(head, sizeof head, "{\"id\": %llu, \"arrival\": %.17g, \"accurate\": {\"encoding\": \"%s\", ",
                    (unsigned long long)th->request_ids[r], arrival ? arrival[r] : 0.0, bitmap ? "bitmap" : "list");
      line = head;
      line += "\"size\": " + std::to_string(S) + ", ";
      const uint32_t* m = idx.data() + offsets[i];
      const uint64_t c = offsets[i + 1] - offsets[i];
      if (bitmap) {
        std::vector<uint8_t> bytes((size_t)((S + 7) / 8), 0);
        for (uint64_t k = 0; k < c; ++k) bytes[m[k] >> 3] |= (uint8_t)(1u << (m[k] & 7));
        static const char* hx = "0123456789abcdef";
        line += "\"bits\": \"";
        for (uint8_t b : bytes) {
          line += hx[b >> 4];
          line += hx[b & 15];
        }
        line += "\"}}\n";
      } else {
        line += "\"members\": [";
        for (uint64_t k = 0; k < c; ++k) {
          if (k) line += ", ";
          line += std::to_string(m[k]);
        }
        line += "]}}\n";
      }
      if (std::fwrite(line.data(), 1, line.size(), f) != line.size()) {
        rc = fail(AG_ERR_IO, std::string("short write to trace file: ") + path);
        break;
      }
      written += line.size();
    }
  }
  if (std::fclose(f) != 0 && rc == AG_OK) rc = fail(AG_ERR_IO, std::string("cannot close trace file: ") + path);
  if (bytes_written) *bytes_written = written;
  return rc;
}
