// Cost of one synchronization step: atomic grid barrier over N co-resident
// CTAs (cooperative launch) vs the hardware cluster barrier (<= 16 CTAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/barrier_probe tools/barrier_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks, unsigned& my_gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned g = my_gen;
    if (atomicAdd(count, 1u) == nblocks - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicExch(gen, g + 1);
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
      } while (cur == g);
    }
    my_gen = g + 1;
    __threadfence();
  }
  __syncthreads();
}

__global__ void grid_k(unsigned* bar, int iters) {
  unsigned my_gen = 0;
  if (threadIdx.x == 0) my_gen = *reinterpret_cast<volatile unsigned*>(bar + 1);
  __syncthreads();
  for (int i = 0; i < iters; ++i) grid_barrier(bar, bar + 1, gridDim.x, my_gen);
}

__global__ void cluster_k(int iters) {
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

int main() {
  unsigned* bar;
  cudaMalloc(&bar, 8);
  cudaMemset(bar, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int nb : {16, 32, 64, 128, 148}) {
    void* args[] = {&bar, (void*)&iters};
    int it = iters;
    args[1] = &it;
    cudaLaunchCooperativeKernel((void*)grid_k, nb, 256, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)grid_k, nb, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid barrier  %3d CTAs: %.3f us/barrier (%s)\n", nb, 1000.0 * ms / iters, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(cluster_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, cluster_k, iters);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, cluster_k, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster barrier %2d CTAs: %.3f us/barrier (%s)\n", cs, 1000.0 * ms / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
