// Launch counter and live per-launch CUDA-event profiler.
//
// Every kernel wrapper bumps a process-wide launch counter (bench.py reports
// it as gpu_launches).  When profiling is on, the executor brackets each
// launch with a pair of pooled CUDA events on the launching stream and tags it
// with a category plus its algorithmic FLOPs / bytes; rgb_profile_collect()
// turns the pairs into per-category device time (bench.py's roofline numbers).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rgb {

enum ProfCat : int {
  PROF_EW = 0,          // elementwise chains over a whole chunk/window
  PROF_GEMM = 1,        // hoisted grouped GEMM (+ fused epilogue)
  PROF_GEMM_FRAME = 2,  // per-frame recurrent GEMM inside an SCC loop
  PROF_EW_FRAME = 3,    // per-frame elementwise chain inside an SCC loop
  PROF_DW = 4,          // grouped weight-gradient GEMM
  PROF_SOFTMAX = 5,
  PROF_INJECT = 6,      // softmax-xent inject + loss
  PROF_SGD = 7,
  PROF_TRANSPOSE = 8,
  PROF_SCC = 9,         // persistent SCC kernel (whole time loop)
  PROF_NCAT = 10
};

void note_launch();
int64_t launch_count();

bool prof_enabled();
int prof_start(cudaStream_t s);  // -1 when off
void prof_stop(int slot, cudaStream_t s, int cat, double flops, double bytes);

}  // namespace rgb
