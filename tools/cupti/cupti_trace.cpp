// Minimal CUPTI activity tracer (the nsys-equivalent this image lacks): kernel start/end
// timestamps per stream, without perturbing the launches.  Loaded by tools/trace_move.py via
// ctypes: ct_start() before the traced call, ct_stop(path) after it writes one JSON line per
// kernel (name, stream, start/end in ms relative to the first kernel).
//   g++ -O2 -shared -fPIC tools/cupti/cupti_trace.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcupti -o tools/cupti/libcupti_trace.so
#include <cupti.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

namespace {
struct Rec {
  std::string name;
  uint32_t stream;
  uint64_t start, end;
  int grid;
};
std::vector<Rec> g_recs;

void CUPTIAPI buffer_requested(uint8_t** buffer, size_t* size, size_t* max_records) {
  *size = 16 * 1024 * 1024;
  *buffer = static_cast<uint8_t*>(aligned_alloc(8, *size));
  *max_records = 0;
}

void CUPTIAPI buffer_completed(CUcontext, uint32_t, uint8_t* buffer, size_t, size_t valid) {
  CUpti_Activity* rec = nullptr;
  while (cuptiActivityGetNextRecord(buffer, valid, &rec) == CUPTI_SUCCESS) {
    if (rec->kind == CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL || rec->kind == CUPTI_ACTIVITY_KIND_KERNEL) {
      auto* k = reinterpret_cast<CUpti_ActivityKernel9*>(rec);
      g_recs.push_back({k->name ? k->name : "?", k->streamId, k->start, k->end,
                        (int)(k->gridX * k->gridY * k->gridZ)});
    }
  }
  free(buffer);
}
}  // namespace

extern "C" {
int ct_start() {
  g_recs.clear();
  if (cuptiActivityRegisterCallbacks(buffer_requested, buffer_completed) != CUPTI_SUCCESS) return 1;
  if (cuptiActivityEnable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL) != CUPTI_SUCCESS) return 2;
  return 0;
}
int ct_stop(const char* path) {
  cuptiActivityFlushAll(1);
  cuptiActivityDisable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
  FILE* f = std::fopen(path, "w");
  if (!f) return 1;
  uint64_t t0 = UINT64_MAX;
  for (auto& r : g_recs) t0 = r.start < t0 ? r.start : t0;
  for (auto& r : g_recs)
    std::fprintf(f, "{\"k\": \"%.80s\", \"s\": %u, \"t0\": %.4f, \"t1\": %.4f, \"grid\": %d}\n", r.name.c_str(), r.stream,
                 (r.start - t0) * 1e-6, (r.end - t0) * 1e-6, r.grid);
  std::fclose(f);
  return (int)g_recs.size();
}
}
