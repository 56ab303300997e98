// Launch counter + pooled-event profiler (see rgb_prof.cuh) and its C ABI.
#include <atomic>
#include <cstring>
#include <vector>

#include "../../include/rnngraph_b200.h"
#include "rgb_prof.cuh"

namespace rgb {
namespace {

std::atomic<int64_t> g_launches{0};

struct Pending {
  int cat;
  double flops, bytes;
};

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // 2 per slot
  std::vector<Pending> pend;
  int used = 0;
  double ms[PROF_NCAT] = {}, flops[PROF_NCAT] = {}, bytes[PROF_NCAT] = {};
  int64_t n[PROF_NCAT] = {};

  void ensure_pool() {
    if (!ev.empty()) return;
    const int slots = 16384;
    ev.resize(2 * slots);
    pend.resize(slots);
    for (auto& e : ev) cudaEventCreate(&e);
  }
  void collect() {
    if (used == 0) return;
    cudaEventSynchronize(ev[2 * (used - 1) + 1]);
    for (int i = 0; i < used; ++i) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]) != cudaSuccess) continue;
      const Pending& p = pend[i];
      ms[p.cat] += t;
      flops[p.cat] += p.flops;
      bytes[p.cat] += p.bytes;
      n[p.cat] += 1;
    }
    used = 0;
  }
};

Profiler g_prof;

}  // namespace

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }
bool prof_enabled() { return g_prof.on; }

int prof_start(cudaStream_t s) {
  if (!g_prof.on) return -1;
  if (g_prof.used * 2 >= (int)g_prof.ev.size()) g_prof.collect();
  const int slot = g_prof.used++;
  cudaEventRecord(g_prof.ev[2 * slot], s);
  return slot;
}

void prof_stop(int slot, cudaStream_t s, int cat, double flops, double bytes) {
  if (slot < 0) return;
  cudaEventRecord(g_prof.ev[2 * slot + 1], s);
  g_prof.pend[slot] = Pending{cat, flops, bytes};
}

}  // namespace rgb

extern "C" {

int rgb_launch_count(int64_t* n) {
  if (!n) return RGB_ERR_KERNEL;
  *n = rgb::launch_count();
  return RGB_OK;
}

int rgb_profile_enable(int on) {
  if (on) rgb::g_prof.ensure_pool();
  else rgb::g_prof.collect();
  rgb::g_prof.on = on != 0;
  return RGB_OK;
}

int rgb_profile_collect(void) {
  rgb::g_prof.collect();
  return cudaGetLastError() == cudaSuccess ? RGB_OK : RGB_ERR_CUDA;
}

int rgb_profile_reset(void) {
  rgb::g_prof.collect();
  std::memset(rgb::g_prof.ms, 0, sizeof rgb::g_prof.ms);
  std::memset(rgb::g_prof.flops, 0, sizeof rgb::g_prof.flops);
  std::memset(rgb::g_prof.bytes, 0, sizeof rgb::g_prof.bytes);
  std::memset(rgb::g_prof.n, 0, sizeof rgb::g_prof.n);
  return RGB_OK;
}

int rgb_profile_read(int cat, double* ms, int64_t* launches, double* flops, double* bytes) {
  if (cat < 0 || cat >= rgb::PROF_NCAT || !ms || !launches || !flops || !bytes) return RGB_ERR_KERNEL;
  *ms = rgb::g_prof.ms[cat];
  *launches = rgb::g_prof.n[cat];
  *flops = rgb::g_prof.flops[cat];
  *bytes = rgb::g_prof.bytes[cat];
  return RGB_OK;
}

}  // extern "C"
