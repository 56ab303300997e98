// tcgen05 kind::tf32 SS-MMA throughput probe (tuning aid, not part of the library).
//
// One CTA per SM; one thread issues `iters` x 12 MMAs (128 x N x 8, operands
// from shared memory, SWIZZLE_128B K-major descriptors over a zeroed 32-deep
// stage) into a TMEM accumulator, committing each group of 12 to an mbarrier.
// Optionally 8 other warps stream LDS.128/STS.128 over a separate smem region
// at the same time (the converter traffic of the GEMM kernels).  Reports MMA
// cycles per group vs the 12 * 128 * N / 256 cycle issue floor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N>
__global__ void __launch_bounds__(288, 1) probe(int iters, int stream_smem, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* a = sm;                      // 16 KB
  uint8_t* b = sm + 16384;              // N * 128 B
  uint8_t* scratch = b + N * 128;       // 64 KB streamed by the other warps
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    stop = 0;
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 8) {
    if ((threadIdx.x & 31) == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        for (int j = 0; j < 4; ++j) {
          const uint64_t da = desc(su32(a) + j * 32), db = desc(su32(b) + j * 32);
          for (int q = 0; q < 3; ++q)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(da), "l"(db), "r"(idesc), "r"(1));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"(su32(&bar)) : "memory");
      out[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (stream_smem) {
    // converter-like traffic: read a float4, write its neighbour
    float4* s4 = reinterpret_cast<float4*>(scratch);
    float acc = 0.f;
    while (!stop) {
      for (int q = threadIdx.x; q < 2048; q += 256) {
        float4 v = s4[q];
        acc += v.x;
        s4[q + 2048] = v;
      }
    }
    if (acc == 1234.f) out[0] = 0;
  }
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int N>
void run(int stream_smem) {
  const int smem = 16384 + N * 128 + 65536 + 1024;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* out;
  cudaMalloc(&out, 148 * 8);
  const int iters = 2000;
  probe<N><<<148, 288, smem>>>(iters, stream_smem, out);
  probe<N><<<148, 288, smem>>>(iters, stream_smem, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  long long h[148];
  cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
  const double per = mean / iters, floor = 12.0 * 128 * N / 256;
  printf("N=%3d smem-stream=%d: %.0f cyc per 12 MMAs (floor %.0f, %.2fx); operand bytes %.0f B/clk\n", N, stream_smem,
         per, floor, per / floor, 12.0 * (128 + N) * 32 / per);
  cudaFree(out);
}

int main() {
  run<256>(0);
  run<256>(1);
  run<128>(0);
  run<128>(1);
  run<64>(0);
  return 0;
}
