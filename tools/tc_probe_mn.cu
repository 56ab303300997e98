// Probe: MN-major tf32 UMMA operands loaded by TMA.
// G[M=128][N=64] = E^T Y with E [K=32][M] and Y [K][N] both MN-contiguous.
// TMA boxes {32 mn (128 B), 32 k} with a 128-byte swizzle variant; UMMA
// descriptor layout type and LBO/SBO variants are tried.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe_mn tools/tc_probe_mn.cu
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

struct Maps { CUtensorMap e, y; };

template <int M, int N, int K>
__global__ void probe(const __grid_constant__ Maps maps, float* G, int layout, uint32_t lbo, uint32_t sbo, uint32_t kstep) {
  __shared__ __align__(1024) float sa[M * K];
  __shared__ __align__(1024) float sb[N * K];
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t bytes = (M + N) * K * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes));
    for (int b = 0; b < M / 32; ++b)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sa) + b * 32 * K * 4), "l"(&maps.e), "r"(b * 32), "r"(0), "r"(su32(&bar)) : "memory");
    for (int b = 0; b < N / 32; ++b)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sb) + b * 32 * K * 4), "l"(&maps.y), "r"(b * 32), "r"(0), "r"(su32(&bar)) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}\n"
                   : "=r"(done) : "r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < K / 8; ++j) {
      const uint64_t da = sdesc(su32(sa) + j * kstep, lbo, sbo, layout);
      const uint64_t db = sdesc(su32(sb) + j * kstep, lbo, sbo, layout);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)(j > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}\n"
                   : "=r"(done) : "r"(su32(&bar2)));
  }
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),
          "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 16; ++i) G[(warp * 32 + lane) * N + c + i] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  constexpr int M = 128, N = 64, K = 32;
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  std::vector<float> E(K * M), Y(K * N), G(M * N), R(M * N);
  srand(3);
  for (auto& v : E) v = (float)((rand() % 17) - 8);
  for (auto& v : Y) v = (float)((rand() % 13) - 6);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)E[k * M + m] * Y[k * N + n];
      R[m * N + n] = (float)s;
    }
  float *dE, *dY, *dG;
  cudaMalloc(&dE, E.size() * 4); cudaMalloc(&dY, Y.size() * 4); cudaMalloc(&dG, G.size() * 4);
  cudaMemcpy(dE, E.data(), E.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  struct V { const char* name; CUtensorMapSwizzle sw; int layout; uint32_t lbo, sbo, kstep; };
  V vs[] = {
      {"ATOM_32B L1 lbo=4096 sbo=512 k+1024", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 1, 4096, 512, 1024},
      {"ATOM_32B L1 lbo=512 sbo=4096 k+1024", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 1, 512, 4096, 1024},
      {"ATOM_32B L1 lbo=4096 sbo=1024 k+1024", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 1, 4096, 1024, 1024},
      {"SW128 L2 lbo=4096 sbo=1024 k+1024", CU_TENSOR_MAP_SWIZZLE_128B, 2, 4096, 1024, 1024},
      {"SW128 L2 lbo=1024 sbo=4096 k+1024", CU_TENSOR_MAP_SWIZZLE_128B, 2, 1024, 4096, 1024},
      {"ATOM_32B L2 lbo=4096 sbo=512 k+1024", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, 2, 4096, 512, 1024},
  };
  for (auto& v : vs) {
    Maps maps;
    cuuint64_t de[2] = {(cuuint64_t)M, (cuuint64_t)K}, dy[2] = {(cuuint64_t)N, (cuuint64_t)K};
    cuuint64_t se[1] = {(cuuint64_t)M * 4}, sy[1] = {(cuuint64_t)N * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult r1 = enc(&maps.e, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dE, de, se, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&maps.y, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dY, dy, sy, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemset(dG, 0xff, G.size() * 4);
    probe<M, N, K><<<1, 128>>>(maps, dG, v.layout, v.lbo, v.sbo, v.kstep);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(G.data(), dG, G.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double err = 0, mx = 0;
    for (int i = 0; i < M * N; ++i) {
      double d = fabs((double)G[i] - R[i]);
      if (!(d < 1e-3)) ++bad;
      err = fmax(err, d);
      mx = fmax(mx, fabs((double)G[i]));
    }
    printf("%-40s enc=%d/%d %s bad=%d max|err|=%g max|G|=%g  G0=%g ref0=%g\n", v.name, (int)r1, (int)r2,
           cudaGetErrorString(e), bad, err, mx, G[0], R[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
