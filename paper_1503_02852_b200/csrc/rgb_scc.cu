// Persistent recurrent-SCC kernel (paper §3.1: the frame-sequential part).
//
// One cooperative launch runs a whole per-frame loop of one strongly connected
// component -- forward (ascending) or backward (descending) -- instead of one or
// two launches per frame.  The loop body is the same int32 step program the
// host executor interprets (schedule.py), copied to shared memory and walked
// by the device every frame:
//   * GEMM step (the intra-SCC dense edges, e.g. cell(t-1) -> {in,forget}
//     gates): CTA b owns output columns [b*W/G, (b+1)*W/G) of every job; the
//     matching rows of the recurrent weights (W_rec) are loaded into shared
//     memory ONCE at kernel start and stay resident for all frames; one warp
//     per (stream, column) dot product, then the fused elementwise epilogue
//     (activation, gates, cell update, f', eps) for that element;
//   * elementwise step: the CTA's own columns (element-local by construction);
//   * a grid barrier precedes every GEMM step -- the only place a CTA reads
//     columns other CTAs wrote (the delayed or zero-delay dense edges).
// Reference semantics: engine.py:405-413 (forward), 568-576 (backward).
#include <cuda_runtime.h>

#include <cstdint>

#include "rgb_ew.cuh"
#include "rgb_kernels.cuh"
#include "rgb_scc.cuh"

namespace rgb {
namespace {

constexpr int kSccThreads = 256;
enum { S_EW = 1, S_GEMM = 2 };

__device__ __forceinline__ long long pmod_d(long long a, long long m) { return ((a % m) + m) % m; }

__device__ __forceinline__ float* resolve_d(const SccCtx& c, int buf, int shift, long long t) {
  const SccBuf b = c.bufs[buf];
  const long long tt = t + shift;
  long long idx;
  if (b.kind == 0) idx = pmod_d(tt, c.cap);
  else if (b.kind == 1) idx = tt - c.t1 + c.hmax - 1;
  else idx = tt - c.chunk_base;
  return c.ws + b.off + idx * (long long)c.S * b.width;
}

// Parse one op (same word layout as rgb_plan.cu parse_op) for frame t.
__device__ int parse_op_d(const int32_t* w, int pos, const SccCtx& c, long long t, EwOp& op) {
  op.kind = w[pos++];
  op.act = w[pos++];
  const int out_buf = w[pos++];
  op.out = resolve_d(c, out_buf, 0, t);
  op.out_is_ring = c.bufs[out_buf].kind == 0;
  op.nterm = w[pos++];
  for (int i = 0; i < op.nterm; ++i, pos += 2) op.term[i] = resolve_d(c, w[pos], w[pos + 1], t);
  op.nrank1 = w[pos++];
  for (int i = 0; i < op.nrank1; ++i, pos += 3) {
    op.r1src[i] = resolve_d(c, w[pos], w[pos + 1], t);
    op.r1w[i] = c.w + c.wts[w[pos + 2]].off;
  }
  op.nfac = w[pos++];
  for (int i = 0; i < op.nfac; ++i, pos += 2) op.fac[i] = resolve_d(c, w[pos], w[pos + 1], t);
  op.y = w[pos] >= 0 ? resolve_d(c, w[pos], w[pos + 1], t) : nullptr;
  pos += 2;
  op.base = w[pos] >= 0 ? resolve_d(c, w[pos], w[pos + 1], t) : nullptr;  // -2 (accumulator) -> null
  pos += 2;
  const int inj = w[pos++];
  op.inj = nullptr;
  op.inj_row0 = 0;
  if (inj && t > c.t0) op.inj = resolve_d(c, c.inj_buf, 0, t);
  const int neps = w[pos++];
  for (int i = 0; i < kMaxFac; ++i) op.eps[i] = nullptr;
  for (int i = 0; i < neps; ++i, ++pos) op.eps[i] = w[pos] >= 0 ? resolve_d(c, w[pos], 0, t) : nullptr;
  return pos;
}

__device__ int parse_chain_d(const int32_t* w, int pos, const SccCtx& c, long long t, EwChain& ch) {
  ch.width = w[pos++];
  ch.nops = w[pos++];
  for (int k = 0; k < ch.nops; ++k) pos = parse_op_d(w, pos, c, t, ch.op[k]);
  return pos;
}

// Skip an op / chain without resolving (used by the weight preload walk).
__device__ int skip_op(const int32_t* w, int pos) {
  pos += 3;
  pos += 1 + 2 * w[pos];
  pos += 1 + 3 * w[pos];
  pos += 1 + 2 * w[pos];
  pos += 4;
  pos += 1;
  pos += 1 + w[pos];
  return pos;
}

__device__ int skip_chain(const int32_t* w, int pos) {
  const int nops = w[pos + 1];
  pos += 2;
  for (int k = 0; k < nops; ++k) pos = skip_op(w, pos);
  return pos;
}

// Sense-reversing grid barrier over the co-resident CTAs of a cooperative launch.
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

struct SJob {
  int nseg, n;
  const float* a[kMaxSegs];
  const float* bs[kMaxSegs];  // weight rows of this CTA's columns (shared or global)
  int k[kMaxSegs];
  int b_ld[kMaxSegs];         // leading dimension of bs (k when cached, k as well in global)
};

__global__ void __launch_bounds__(kSccThreads, 1) scc_kernel(const __grid_constant__ SccCtx c) {
  extern __shared__ __align__(16) unsigned char sm[];
  int32_t* words = reinterpret_cast<int32_t*>(sm);
  const int words_pad = (c.body_len + 3) & ~3;
  float* wcache = reinterpret_cast<float*>(words + words_pad);
  SJob* jobs = reinterpret_cast<SJob*>(wcache + ((c.wcache_floats + 3) & ~3LL));  // 16-B aligned
  EwChain* chains = reinterpret_cast<EwChain*>(jobs + kMaxJobs);
  __shared__ int s_nunits;

  for (int i = threadIdx.x; i < c.body_len; i += blockDim.x) words[i] = c.body[i];
  const int W = c.width;
  const int j0 = (int)((long long)blockIdx.x * W / gridDim.x);
  const int j1 = (int)((long long)(blockIdx.x + 1) * W / gridDim.x);
  const int ncol = j1 - j0;
  __syncthreads();

  // preload this CTA's weight rows of every GEMM step (identical walk in all threads)
  if (c.use_cache) {
    int pos = 0, off = 0;
    while (pos < c.body_len) {
      const int kind = words[pos++];
      if (kind == S_GEMM) {
        const int njobs = words[pos++];
        for (int jb = 0; jb < njobs; ++jb) {
          const int nseg = words[pos++];
          for (int s = 0; s < nseg; ++s, pos += 4) {
            const int cid = words[pos + 2], trans = words[pos + 3];
            const SccW wd = c.wts[cid];
            const int K = trans ? wd.rows : wd.cols;
            const float* src = (trans ? c.wt : c.w) + wd.off + (long long)j0 * K;
            for (int i = threadIdx.x; i < ncol * K; i += blockDim.x) wcache[off + i] = src[i];
            off += ncol * K;
          }
          pos = skip_chain(words, pos);
        }
      } else {
        const int nch = words[pos++];
        for (int i = 0; i < nch; ++i) pos = skip_chain(words, pos);
      }
    }
  }
  unsigned my_gen = 0;
  if (threadIdx.x == 0) my_gen = *reinterpret_cast<volatile unsigned*>(c.bar + 1);
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int f = 0; f < c.frames; ++f) {
    const long long t = c.reverse ? c.t_first + c.frames - 1 - f : c.t_first + f;
    RingWrite ring;
    ring.split = (long long)(c.cap - pmod_d(t, c.cap)) * c.S;
    ring.frame_rows = (long long)c.cap * c.S;
    int pos = 0, woff = 0;
    while (pos < c.body_len) {
      const int kind = words[pos];
      if (kind == S_GEMM) {
        grid_barrier(c.bar, c.bar + 1, gridDim.x, my_gen);
        const int njobs = words[pos + 1];
        if (threadIdx.x == 0) {
          int p = pos + 2;
          for (int jb = 0; jb < njobs; ++jb) {
            SJob& J = jobs[jb];
            J.nseg = words[p++];
            for (int s = 0; s < J.nseg; ++s, p += 4) {
              const int ab = words[p], ash = words[p + 1], cid = words[p + 2], trans = words[p + 3];
              const SccW wd = c.wts[cid];
              const int K = trans ? wd.rows : wd.cols;
              J.a[s] = resolve_d(c, ab, ash, t);
              J.k[s] = K;
              J.b_ld[s] = K;
              if (c.use_cache) {
                J.bs[s] = wcache + woff;
                woff += ncol * K;
              } else {
                J.bs[s] = (trans ? c.wt : c.w) + wd.off + (long long)j0 * K;
              }
            }
            p = parse_chain_d(words, p, c, t, chains[jb]);
            J.n = chains[jb].width;
          }
          s_nunits = p;  // end of the step
        }
        __syncthreads();
        pos = s_nunits;  // (woff is only meaningful in thread 0, which resolved the pointers)
        // one warp per (job, stream, column): dot products over all segments
        const int items = njobs * c.S * ncol;
        for (int it = warp; it < items; it += nwarps) {
          const int jb = it / (c.S * ncol), rem = it - jb * (c.S * ncol);
          const int srow = rem / ncol, col = rem - srow * ncol;
          const SJob& J = jobs[jb];
          float acc = 0.f;
          for (int s = 0; s < J.nseg; ++s) {
            const float* a = J.a[s] + (long long)srow * J.k[s];
            const float* b = J.bs[s] + (long long)col * J.b_ld[s];
            for (int k = lane; k < J.k[s]; k += 32) acc = fmaf(a[k], b[k], acc);
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) {
            const EwChain& ch = chains[jb];
            for (int k = 0; k < ch.nops; ++k) ew_apply(ch.op[k], ch.width, srow, j0 + col, ring, k == 0, acc);
          }
        }
        __syncthreads();
      } else {  // S_EW
        const int nch = words[pos + 1];
        if (threadIdx.x == 0) {
          int p = pos + 2;
          for (int i = 0; i < nch; ++i) p = parse_chain_d(words, p, c, t, chains[i]);
          s_nunits = p;
        }
        __syncthreads();
        pos = s_nunits;
        for (int i = 0; i < nch; ++i) {
          const EwChain& ch = chains[i];
          const int items = c.S * ncol;
          for (int e = threadIdx.x; e < items; e += blockDim.x) {
            const int srow = e / ncol, col = j0 + (e - (e / ncol) * ncol);
            for (int k = 0; k < ch.nops; ++k) ew_apply(ch.op[k], ch.width, srow, col, ring, false, 0.0f);
          }
        }
        __syncthreads();
      }
    }
  }
}

}  // namespace

size_t scc_smem_bytes(int body_len, long long wcache_floats) {
  static_assert(sizeof(SJob) % 16 == 0 || sizeof(SJob) % 8 == 0, "SJob keeps 8-byte alignment");
  return (size_t)((body_len + 3) & ~3) * 4 + (size_t)((wcache_floats + 3) & ~3LL) * 4 + sizeof(SJob) * kMaxJobs +
         sizeof(EwChain) * kMaxChains + 64;
}

int scc_max_blocks(size_t smem) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaFuncSetAttribute(scc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scc_kernel, kSccThreads, smem) != cudaSuccess) return 0;
  return per_sm * sms;
}

cudaError_t launch_scc(const SccCtx& c, int blocks, size_t smem, cudaStream_t s) {
  // the attribute is per function, not per launch: (re)set it for this size
  cudaError_t e = cudaFuncSetAttribute(scc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<SccCtx*>(&c)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(scc_kernel), dim3(blocks), dim3(kSccThreads), args,
                                     smem, s);
}

}  // namespace rgb
