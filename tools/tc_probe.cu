// Standalone probe of tcgen05.mma kind::tf32 smem-descriptor variants (K-major vs
// MN-major operands, LBO/SBO assignments).  One CTA, M=128, N=64, K=8..32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cstring>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// A: [M=128][K] row-major global, B: [N=64][K] row-major global, C = A B^T.
// smem layouts: K-major SW128 (rows of 32 fp32) or MN-major SW128 atoms [8 k][32 mn].
template <int M, int N, int K>
__global__ void probe(const float* A, const float* B, float* C, int a_mn, int b_mn, int variant) {
  __shared__ __align__(1024) float sa[M * 32];
  __shared__ __align__(1024) float sb[N * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  // fill (K <= 32): element (r, k)
  for (int i = tid; i < M * 32; i += blockDim.x) {
    int r = i / 32, k = i % 32;
    float v = k < K ? A[r * K + k] : 0.f;
    int byte;
    if (!a_mn) byte = r * 128 + ((((k >> 2) ^ (r & 7))) << 4) + (k & 3) * 4;
    else byte = ((k >> 3) * (M / 32) + (r >> 5)) * 1024 + (k & 7) * 128 + ((((r & 31) >> 2) ^ (k & 7)) << 4) + (r & 3) * 4;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(sa) + byte) = v;
  }
  for (int i = tid; i < N * 32; i += blockDim.x) {
    int r = i / 32, k = i % 32;
    float v = k < K ? B[r * K + k] : 0.f;
    int byte;
    if (!b_mn) byte = r * 128 + ((((k >> 2) ^ (r & 7))) << 4) + (k & 3) * 4;
    else byte = ((k >> 3) * (N / 32) + (r >> 5)) * 1024 + (k & 7) * 128 + ((((r & 31) >> 2) ^ (k & 7)) << 4) + (r & 3) * 4;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(sb) + byte) = v;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < (K + 7) / 8; ++j) {
      uint32_t ao, bo, albo, asbo, blbo, bsbo;
      if (!a_mn) { ao = j * 32; albo = 16; asbo = 1024; }
      else {
        ao = j * (M / 32) * 1024;
        if (variant == 0) { albo = 1024; asbo = (M / 32) * 1024; } else { albo = (M / 32) * 1024; asbo = 1024; }
      }
      if (!b_mn) { bo = j * 32; blbo = 16; bsbo = 1024; }
      else {
        bo = j * (N / 32) * 1024;
        if (variant == 0) { blbo = 1024; bsbo = (N / 32) * 1024; } else { blbo = (N / 32) * 1024; bsbo = 1024; }
      }
      uint64_t da = sdesc(smem_u32(sa) + ao, albo, asbo, 2), db = sdesc(smem_u32(sb) + bo, blbo, bsbo, 2);
      uint32_t acc = j > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),
          "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 16; ++i) C[(warp * 32 + lane) * N + c + i] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

// How does kind::tf32 consume the low 13 mantissa bits of an fp32 operand?
// A = x (row 0), B = identity-like column e0 -> C[0][0] = tf32view(x).
void rounding_probe() {
  constexpr int M = 128, N = 64, K = 32;
  std::vector<float> A(M * K, 0.f), B(N * K, 0.f), C(M * N);
  const float xs[6] = {1.0f + 0x1p-12f, 1.0f + 3 * 0x1p-12f, 1.0f + 0x1p-11f, 1.0f + 0x1.8p-11f,
                       1.0f + 5 * 0x1p-13f, -(1.0f + 3 * 0x1p-12f)};
  for (int i = 0; i < 6; ++i) A[i * K + 0] = xs[i];
  B[0 * K + 0] = 1.0f;
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  probe<M, N, K><<<1, 256>>>(dA, dB, dC, 0, 0, 0);
  cudaDeviceSynchronize();
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 6; ++i) {
    float x = xs[i];
    uint32_t u; memcpy(&u, &x, 4);
    uint32_t t = u & 0xFFFFE000u; float tr; memcpy(&tr, &t, 4);
    printf("x=%.10f  mma=%.10f  trunc=%.10f  %s\n", x, C[i * N + 0], tr, C[i * N] == tr ? "TRUNCATES" : "rounds");
  }
}

int main() {
  rounding_probe();
  constexpr int M = 128, N = 64, K = 32;
  std::vector<float> A(M * K), B(N * K), C(M * N), R(M * N);
  srand(1);
  for (auto& v : A) v = (float)((rand() % 17) - 8);  // small integers: exact in tf32
  for (auto& v : B) v = (float)((rand() % 13) - 6);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      R[i * N + j] = (float)s;
    }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int a_mn = 0; a_mn < 2; ++a_mn)
    for (int b_mn = 0; b_mn < 2; ++b_mn)
      for (int variant = 0; variant < 2; ++variant) {
        if (!a_mn && !b_mn && variant) continue;
        cudaMemset(dC, 0xff, C.size() * 4);
        probe<M, N, K><<<1, 256>>>(dA, dB, dC, a_mn, b_mn, variant);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        int bad = 0;
        for (int i = 0; i < M * N; ++i) {
          double d = fabs((double)C[i] - R[i]);
          if (!(d < 1e-3)) ++bad;
          err = fmax(err, d);
          mx = fmax(mx, fabs((double)C[i]));
        }
        printf("a_mn=%d b_mn=%d variant=%d: %s max|err|=%g max|C|=%g bad=%d  C[0..3]=%g %g %g %g ref=%g %g %g %g\n", a_mn,
               b_mn, variant, cudaGetErrorString(e), err, mx, bad, C[0], C[1], C[2], C[3], R[0], R[1], R[2], R[3]);
      }
  return 0;
}
