// TMA load-throughput probe (tuning aid, not part of the library).
//
// One CTA per SM, one thread issues 2-D tiled TMA loads of an L2-resident
// fp32 matrix into a ring of smem stages and waits on each stage's mbarrier
// before reusing it.  Reports bytes/clk/SM and the issue-to-issue gap for
//   - tensor map passed as a __grid_constant__ kernel parameter vs read from
//     global memory (the library keeps its maps in a device table);
//   - box {16 fp32, R} SWIZZLE_64B vs {32 fp32, R} SWIZZLE_128B;
//   - stages in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool PARAM>
__global__ void __launch_bounds__(512, 1) probe(const __grid_constant__ CUtensorMap pm, const CUtensorMap* gm,
                                                int iters, int stages, int stage_bytes, int box_w, int box_h,
                                                int rows, int cols, long long* out, int prefetch, int stream_warps) {
  extern __shared__ __align__(1024) uint8_t sm_base[];
  uint8_t* sm = sm_base;
  const int nw = blockDim.x / 32 - stream_warps, w = threadIdx.x / 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm_base + nw * stages * stage_bytes) + w * stages;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (w >= nw) {
    // converter-like smem traffic over a 64 KB region after the barriers
    float4* s4 = reinterpret_cast<float4*>(sm_base + nw * stages * stage_bytes + 1024);
    float acc = 0.f;
    while (!stop) {
      for (int q = threadIdx.x - nw * 32; q < 2048; q += stream_warps * 32) {
        float4 v = s4[q];
        acc += v.x;
        s4[q + 2048] = v;
      }
    }
    if (acc == 1234.f) out[0] = 0;
    return;
  }
  if ((threadIdx.x & 31) != 0) return;
  sm += w * stages * stage_bytes;
  const CUtensorMap* map = PARAM ? &pm : gm;
  if (prefetch) asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int per_stage = stage_bytes / (box_w * box_h * 4);
  long long t0 = clock64(), tw = 0, ti = 0;
  int x = 0, y = ((blockIdx.x + 37 * w) * 977) % (rows / box_h) * box_h;
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    long long c0 = clock64();
    if (it >= stages) {
      const uint32_t par = ((it / stages) - 1) & 1;
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"(su32(&bar[s])), "r"(par) : "memory");
    }
    long long c1 = clock64();
    tw += c1 - c0;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage_bytes) : "memory");
    for (int b = 0; b < per_stage; ++b) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(sm + s * stage_bytes + b * box_w * box_h * 4)),
          "l"(map), "r"(x), "r"(y), "r"(su32(&bar[s]))
          : "memory");
      y += box_h;
      if (y >= rows) { y = 0; x += box_w; if (x >= cols) x = 0; }
    }
    ti += clock64() - c1;
  }
  for (int s = 0; s < stages; ++s) {
    const int last = iters - stages + s;
    if (last < 0) continue;
    const uint32_t par = (last / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(done) : "r"(su32(&bar[last % stages])), "r"(par) : "memory");
  }
  if (w == 0) {
    stop = 1;
    out[blockIdx.x] = clock64() - t0;
    out[148 + blockIdx.x] = tw;
    out[296 + blockIdx.x] = ti;
  }
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int rows = 4096, cols = 1024;  // 16 MB, L2 resident
  float* a;
  cudaMalloc(&a, (size_t)rows * cols * 4);
  cudaMemset(a, 0, (size_t)rows * cols * 4);
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  long long* out;
  cudaMalloc(&out, 3 * 148 * 8);
  int sms = 148;
  struct Case { int box_w, box_h, stages, stage_kb; bool param; int prefetch; int warps = 1; int stream = 0; };
  Case cases[] = {
      {32, 128, 3, 32, true, 0, 1, 0}, {32, 128, 3, 32, true, 0, 1, 8},
      {32, 256, 3, 32, true, 0, 1, 0}, {32, 256, 3, 32, true, 0, 1, 8},
      {32, 128, 6, 16, true, 0, 1, 0}, {32, 128, 6, 16, true, 0, 1, 8},
  };
  for (const Case& c : cases) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.box_w, (cuuint32_t)c.box_h};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     c.box_w == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
    cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice);
    const int sb = c.stage_kb * 1024, smem = c.warps * c.stages * sb + 1024 + (c.stream ? 65536 + 1024 : 0);
    auto k = c.param ? probe<true> : probe<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    for (int rep = 0; rep < 2; ++rep)
      k<<<sms, 32 * (c.warps + c.stream), smem>>>(m, gm, iters, c.stages, sb, c.box_w, c.box_h, rows, cols, out, c.prefetch, c.stream);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[3 * 148];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    double mx = 0, mean = 0, mw = 0, mi = 0;
    for (int i = 0; i < sms; ++i) {
      mx = h[i] > mx ? h[i] : mx;
      mean += h[i] / (double)sms;
      mw += h[148 + i] / (double)sms / iters;
      mi += h[296 + i] / (double)sms / iters;
    }
    printf("stream %d ", c.stream);
    printf("box {%2d,%3d} %s%s %d warps x stages %2d x %2d KB: %6.1f B/clk/SM (mean cyc/stage %.0f)\n", c.box_w,
           c.box_h, c.param ? "param " : "global", c.prefetch ? "+pf" : "   ", c.warps, c.stages, c.stage_kb,
           (double)iters * sb * c.warps / mean, mean / iters);
    printf("      wait %.0f cyc/stage, issue %.0f cyc/stage\n", mw, mi);
  }
  return 0;
}
