// Gradient exchange helpers shared by the executor (rgb_plan.cu) and the
// NCCL binding (rgb_comm.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

struct rgb_comm;

namespace rgb {
// thread-local rgb_last_error() message (defined in rgb_plan.cu)
void set_last_error(const char* msg);
// in-place SUM of `count` floats over all ranks on stream st (NCCL)
int comm_allreduce_f32(rgb_comm* c, float* g, size_t count, cudaStream_t st);
// ncclGroupStart (start = true) / ncclGroupEnd
int comm_group(bool start);
}  // namespace rgb
