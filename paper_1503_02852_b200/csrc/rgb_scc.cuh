// Persistent recurrent-SCC kernel (rgb_scc.cu): launch descriptor.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "rgb_types.cuh"

namespace rgb {

// threads per CTA of the persistent SCC kernel (12 warps: one chain element
// per thread for up to 384 (stream row, unit) pairs per CTA)
constexpr int kSccThreads = 384;

struct SccBuf {
  int kind, width;
  long long off;
};
struct SccW {
  int rows, cols;
  long long off;
};

struct SccCtx {
  const int32_t* body;      // device copy of the loop-body step words
  int body_len;
  int width;                // common width W of every layer the body writes
  const SccBuf* bufs;       // device copies of the plan's buffer / weight tables
  const SccW* wts;
  int nbufs, nwts;
  float* ws;
  const float* w;
  const float* wt;
  long long t_first;        // first frame of the loop (ascending order)
  int frames, reverse;
  long long t1, t0, chunk_base;
  int S, cap, hmax, maxd;
  int inj_buf, use_cache;
  int cluster;              // 1: one thread-block cluster per row block, hardware cluster barrier
  int ncb, nrb;             // CTAs per row block (column split of W) x row blocks (stream split of S)
  int threads;              // CTA size: 256, or kSccThreads when a CTA owns more than 256 elements
  unsigned char* tcache;    // this loop body's template image (built by the first launch), or null
  long long wcache_floats;  // per-CTA shared-memory weight cache (0 = read W from global)
  long long acc_floats;     // per-CTA accumulator staging
  long long stage_floats;   // per-CTA A-operand staging (0 = read A from global)
  long long arena_bytes;    // per-CTA template arena
  long long vals_floats;    // per-CTA forwarded chain values: vals_cap x vals_stride floats
  int vals_cap, vals_stride;
  unsigned* bar;            // [count, generation] of the grid barrier
};

constexpr int kSccTcacheBytes = 64 * 1024;  // per loop body
bool scc_tcache_fits(long long arena_bytes);
size_t scc_smem_bytes(const SccCtx& c);
size_t scc_arena_bytes(int max_jobs_total, int max_chains_total);
int scc_max_blocks(size_t smem);  // co-resident CTAs for a cooperative launch
int scc_max_clusters(int ncb, size_t smem);  // co-resident clusters of ncb CTAs
cudaError_t launch_scc(const SccCtx& c, int blocks, size_t smem, cudaStream_t s);

}  // namespace rgb
