// tcgen05 grouped GEMMs for sm_100a (5th-gen tensor cores, TMEM accumulators).
//
// fp32-exact mode = 3xTF32: every fp32 operand x is split on the fly into
// hi = tf32(x) and lo = tf32(x - hi); the tile product is accumulated in fp32
// TMEM as hi*hi + hi*lo + lo*hi (the lo*lo term is below fp32 rounding of the
// result), which keeps the normwise error ~1e-6 -- inside the fp32 path's
// 1e-4 bound, unlike single-pass TF32 (~1e-3).
//
// Roles (256 threads, one CTA per output tile, 1 CTA/SM by smem):
//   warps 0-3  producers: coalesced 16-B global loads of the fp32 A/B tiles,
//              split into hi/lo, stored into the 128-byte-swizzled K-major
//              UMMA canonical layout (dW's MN-contiguous operands are
//              transposed while loading, so there is no transpose pass;
//              kind::tf32 with MN-major SW128 descriptors returns zeros on
//              sm_100a -- tools/tc_probe.cu), fence.proxy.async, arrive on
//              the stage's "full" mbarrier;
//   warp 4     one elected thread issues 3 x (BK/8) tcgen05.mma.kind::tf32
//              per stage and tcgen05.commit's the stage back to the
//              producers ("empty"), and the accumulator to the epilogue;
//   warps 0-7  epilogue: tcgen05.ld the accumulator (32x32b.x16) and run the
//              fused elementwise chain (bias, identity terms, activation,
//              f', gate co-factors, eps) or the dW store.
//
// Descriptor bit layouts follow the SM100 UMMA smem / instruction descriptor
// formats (vendored CUTLASS cute/arch/mma_sm100_desc.hpp); all code here is
// hand-written.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>

#include "rgb_ew.cuh"
#include "rgb_kernels.cuh"

namespace rgb {
namespace tc {

// tuning aid: per-stage clock64 trace of CTA 0 (tools/build_exp.sh trace -DRGB_EXP_TRACE)
#ifdef RGB_EXP_TRACE
__device__ long long g_trace[6][1024];
__device__ long long g_cta[1024][6];  // globaltimer: start, mainloop done, epilogue done; smid
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifndef RGB_EXP_TRACE_GRID
#define RGB_EXP_TRACE_GRID 0  // trace only launches of this grid size (0: all)
#endif
#define TRACE_ON (RGB_EXP_TRACE_GRID == 0 || gridDim.x == RGB_EXP_TRACE_GRID)
#define CTA_MARK(i) \
  if (TRACE_ON && threadIdx.x == 0 && blockIdx.x < 1024) g_cta[blockIdx.x][i] = gtimer();
#define TRACE(row, it) \
  if (TRACE_ON && blockIdx.x == 0 && (it) < 1024) g_trace[row][it] = clock64();
#else
#define TRACE(row, it)
#define CTA_MARK(i)
#endif


constexpr int BM = 128;   // UMMA M, cta_group::1
constexpr int BK = 32;    // fp32 per stage along K: one 128-byte swizzle row
constexpr int kThreads = 288;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// SM100 shared-memory matrix descriptor, SWIZZLE_128B, version 1.
// layout 2 = SWIZZLE_128B (K-major operands), 1 = SWIZZLE_128B_BASE32B (the
// MN-major tf32 layout TMA's 128B_ATOM_32B swizzle produces).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (Blackwell)
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B, M x N, majors.
__device__ __forceinline__ uint32_t idesc_tf32(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// 2-D tiled TMA load (box {32 fp32 along the row, R rows}, SWIZZLE_128B) into
// smem, completing `bytes` on the mbarrier.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// i-th tensor map of a table (CUtensorMap is 128 bytes; the tables hold plain
// void pointers so this file does not depend on cuda.h)
__device__ __forceinline__ const void* map_at(const void* table, int i) {
  return static_cast<const uint8_t*>(table) + 128 * i;
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(smem_dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// tf32 residual of an fp32 value: kind::tf32 consumes only the top 19 bits
// (it truncates -- measured, tools/tc_probe.cu), so x itself acts as "hi" and
// lo = x - trunc13(x) is exact in fp32.
__device__ __forceinline__ float tf32_residual(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// x -> tf32_rna(x) over `bytes` of shared memory (plain TF32 mode operands)
__device__ __forceinline__ void round_tf32_inplace(uint8_t* base, int bytes, int tid, int nthreads) {
  float4* v = reinterpret_cast<float4*>(base);
  for (int q = tid; q < bytes / 16; q += nthreads) {
    const float4 x = v[q];
    v[q] = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
  }
}

// One operand tile source: `rows` is the valid extent along M (or N), `kv` the
// valid extent along K, ld the global leading dimension (elements).
struct Src {
  const float* p;
  int64_t ld;
  int rows, kv;
  bool vec;  // 16-byte loads allowed
};

constexpr int kProducers = 256;  // warps 0-7 produce (and run the epilogue); warp 8 issues MMAs

// Two-phase tile producer: every global load of a stage is issued before any
// of them is consumed (one memory latency per stage instead of one per
// chunk), then the fp32 values are split into tf32 hi/lo and stored into the
// 128-byte-swizzled K-major layout: row r at r*128 B, 16-byte chunk c at
// (c ^ (r & 7)).  K-major source: the chunk is one 16-B load; MN-contiguous
// source (dW operands): lanes walk consecutive rows and gather the chunk's four
// k values with coalesced 4-B loads, i.e. the tile is transposed on the fly.
template <int TILE, bool MN_MAJOR>
struct TileLoad {
  static constexpr int NPT = TILE * BK / 4 / kProducers;  // 16-B chunks per producer thread
  float4 v[NPT];

  __device__ __forceinline__ void load(const Src& s, int mn0, int k0, int tid) {
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const int q = tid + i * kProducers;
      int r, c;
      if (!MN_MAJOR) { r = q >> 3; c = q & 7; } else { r = q % TILE; c = q / TILE; }
      const int gr = mn0 + r, gk = k0 + c * 4;
      if (!MN_MAJOR) {
        const float* src = s.p + (int64_t)gr * s.ld + gk;
        if (gr < s.rows && s.vec && gk + 3 < s.kv) {
          v[i] = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          v[i].x = (gr < s.rows && gk + 0 < s.kv) ? src[0] : 0.f;
          v[i].y = (gr < s.rows && gk + 1 < s.kv) ? src[1] : 0.f;
          v[i].z = (gr < s.rows && gk + 2 < s.kv) ? src[2] : 0.f;
          v[i].w = (gr < s.rows && gk + 3 < s.kv) ? src[3] : 0.f;
        }
      } else {
        const float* src = s.p + (int64_t)gk * s.ld + gr;
        const bool ok = gr < s.rows;
        v[i].x = (ok && gk + 0 < s.kv) ? __ldg(src) : 0.f;
        v[i].y = (ok && gk + 1 < s.kv) ? __ldg(src + s.ld) : 0.f;
        v[i].z = (ok && gk + 2 < s.kv) ? __ldg(src + 2 * s.ld) : 0.f;
        v[i].w = (ok && gk + 3 < s.kv) ? __ldg(src + 3 * s.ld) : 0.f;
      }
    }
  }

  __device__ __forceinline__ void store(float* hi, float* lo, int tid) const {
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const int q = tid + i * kProducers;
      int r, c;
      if (!MN_MAJOR) { r = q >> 3; c = q & 7; } else { r = q % TILE; c = q / TILE; }
      const int byte = r * 128 + ((c ^ (r & 7)) << 4);
      float4 h, l;
      h.x = tf32_rna(v[i].x); l.x = tf32_rna(v[i].x - h.x);
      h.y = tf32_rna(v[i].y); l.y = tf32_rna(v[i].y - h.y);
      h.z = tf32_rna(v[i].z); l.z = tf32_rna(v[i].z - h.z);
      h.w = tf32_rna(v[i].w); l.w = tf32_rna(v[i].w - h.w);
      *reinterpret_cast<float4*>(reinterpret_cast<char*>(hi) + byte) = h;
      *reinterpret_cast<float4*>(reinterpret_cast<char*>(lo) + byte) = l;
    }
  }
};

// The job's elementwise chain is copied from the (large, dynamically indexed)
// kernel parameter block into shared memory once per CTA: read per element
// from param space it cost ~0.5 us per 8 elements (indexed constant-cache
// misses), 40% of a 512x4096x1024 launch (tools/gemm_bench.py trace build).
constexpr int kChainBytes = 1280;
static_assert(sizeof(EwChain) <= kChainBytes, "chain staging slot");

__device__ __forceinline__ void stage_chain(EwChain* dst, const EwChain& src, int tid, int nthreads) {
  const int* s = reinterpret_cast<const int*>(&src);
  int* d = reinterpret_cast<int*>(dst);
  for (int i = tid; i < (int)(sizeof(EwChain) / 4); i += nthreads) d[i] = s[i];
}

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN == 256 ? 2 : (BN == 128 ? 3 : (BN == 64 ? 4 : 5));
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + kChainBytes;
  static constexpr int EPI_LD = BN + 4;  // padded staging row (conflict-free 16-B stores)
  static_assert(BM * EPI_LD * 4 <= STAGES * STAGE_BYTES, "epilogue staging must fit in the pipeline smem");
};

__device__ __forceinline__ void find_job(const int* tile_start, int njobs, int bid, int& job, int& tile) {
  job = 0;
  while (job + 1 < njobs && bid >= tile_start[job + 1]) ++job;
  tile = bid - tile_start[job];
}

// Epilogue, run by 256 threads after the accumulator is complete:
// (1) tcgen05.ld the TMEM tile into a padded smem tile (warp w reads lane
//     quarter w%4, column half w/4);
// (2) walk the tile with consecutive threads on consecutive columns and apply
//     the job's elementwise chain (or the dW store) to U elements per thread
//     at a time, gathering every operand of an op for all U before storing.
template <int BN, bool IS_DW, class P>
__device__ __forceinline__ void epilogue(const P& p, int jid, int m0, int n0, int M, int N, uint32_t tmem,
                                         float* tile_s, const EwChain* chain_s, int tid, int tile_lin, int split,
                                         int splits, int r_lo = 0, int r_hi = BM, int phases = 3) {
  using C = Cfg<BN>;
  const int warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int r_loc = quarter * 32 + lane;
  for (int cc = half * (BN / 2); (phases & 1) && cc < (half + 1) * (BN / 2); cc += 16) {
    if (n0 + cc >= N) break;  // warp-uniform
    float v[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cc, v);
    float4* dst = reinterpret_cast<float4*>(tile_s + r_loc * C::EPI_LD + cc);
    dst[0] = make_float4(v[0], v[1], v[2], v[3]);
    dst[1] = make_float4(v[4], v[5], v[6], v[7]);
    dst[2] = make_float4(v[8], v[9], v[10], v[11]);
    dst[3] = make_float4(v[12], v[13], v[14], v[15]);
  }
  if (phases & 1) asm volatile("bar.sync 1, 256;" ::: "memory");
  if (!(phases & 2)) return;  // cluster split-K: the caller reduces the partial tiles first
  if constexpr (!IS_DW) {
    if (splits > 1) {
      // split-K: publish this partial tile and stop; splitk_epilogue_kernel
      // sums the partials in split order (deterministic) and runs the chain
      // with every SM taking part
      constexpr int Q = BM * BN / 4;
      float* part = p.part + ((size_t)tile_lin * splits + split) * (BM * BN);
      for (int q = tid; q < Q; q += 256) {
        const int r = q / (BN / 4), c = (q % (BN / 4)) * 4;
        st4(part, r * BN + c, *reinterpret_cast<const float4*>(tile_s + r * C::EPI_LD + c));
      }
      return;
    }
  }
  const int ncols = (N - n0) < BN ? (N - n0) : BN;
  // local rows [r_lo, nrows) of the tile (a row slice under cluster split-K)
  const int nrows = min((M - m0) < BM ? (M - m0) : BM, r_hi);
  const int total = ncols * max(nrows - r_lo, 0);
  constexpr int U = 8;
  float* g_out = nullptr;
  float alpha = 0.0f;
  RingWrite ring{};
  bool vec;
  if constexpr (IS_DW) {
    g_out = p.job[jid].g;
    alpha = p.alpha;
    vec = N % 4 == 0 && aligned16(g_out);
  } else {
    ring = p.ring;
    vec = chain_vec_ok(*chain_s, N);
  }
  if (vec) {
    // warp-per-row walk: LPR lanes cover one row with 16-byte accesses, each
    // thread takes R = 2 rows per pass (fully coalesced, no index division)
    constexpr int LPR = BN >= 128 ? 32 : BN / 4;  // lanes per row
    constexpr int RPW = 32 / LPR;                  // rows per warp access
    constexpr int CG = BN / 4 / LPR;               // float4 groups per lane per row
#ifndef RGB_EPI_R
#define RGB_EPI_R 4
#endif
    constexpr int R = RGB_EPI_R;  // rows per thread and pass: one operand latency per op covers R rows
    const int sub = lane / LPR, lc = lane % LPR;
#pragma unroll 1
    for (int rb = r_lo + warp * RPW + sub; rb < nrows; rb += 8 * RPW * R) {
#pragma unroll
      for (int g = 0; g < CG; ++g) {
        const int cl = (g * LPR + lc) * 4;
        if (cl >= ncols) continue;
        int64_t rr[R];
        bool ok[R];
        float4 acc[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const int rl = rb + u * 8 * RPW;
          ok[u] = rl < nrows;
          rr[u] = m0 + (ok[u] ? rl : 0);
          acc[u] = *reinterpret_cast<const float4*>(tile_s + (ok[u] ? rl : 0) * C::EPI_LD + cl);
        }
        if constexpr (IS_DW) {
#pragma unroll
          for (int u = 0; u < R; ++u)
            if (ok[u])
              st4(g_out, rr[u] * N + n0 + cl,
                  make_float4(alpha * acc[u].x, alpha * acc[u].y, alpha * acc[u].z, alpha * acc[u].w));
        } else {
          const EwChain& epi = *chain_s;
#ifdef RGB_EXP_TRACE
          if (threadIdx.x == 0) { TRACE(3, 16) }
          for (int k = 0; k < epi.nops; ++k) {
            ew_apply_vec_variant<R>(epi.op[k], N, rr, n0 + cl, ok, ring, k == 0, acc);
            if (threadIdx.x == 0) { TRACE(3, 17 + k) }
          }
#else
          ew_chain_vec<R>(epi, N, rr, n0 + cl, ok, ring, true, acc);
#endif
        }
      }
    }
    return;
  }
#ifdef RGB_EXP_TRACE
  if (tid == 0) { TRACE(3, 15) }
#endif
#pragma unroll 1
  for (int base = 0; base < total; base += 256 * U) {
    int64_t rr[U];
    int cc[U];
    bool ok[U];
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = base + tid + 256 * u;
      ok[u] = idx < total;
      const int rl = r_lo + (ok[u] ? idx / ncols : 0), cl = ok[u] ? idx - (idx / ncols) * ncols : 0;
      rr[u] = m0 + rl;
      cc[u] = n0 + cl;
      acc[u] = tile_s[rl * C::EPI_LD + cl];
    }
    if constexpr (IS_DW) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) g_out[rr[u] * N + cc[u]] = alpha * acc[u];
    } else {
      const EwChain& epi = *chain_s;
      for (int k = 0; k < epi.nops; ++k) ew_apply_batch<U>(epi.op[k], N, rr, cc, ok, ring, k == 0, acc);
    }
  }
}

// IS_DW = false: C[r, n] = sum_seg A_seg[r, :] . B_seg[n, :] (both K-major), EW-chain epilogue.
// IS_DW = true:  G[m, n] = alpha * sum_k E[k, m] Y[k, n] (both MN-contiguous in
//                global memory, K-major in smem), plain store.
template <int BN, bool IS_DW, class P>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(const __grid_constant__ P p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SWIZZLE_128B); offset arithmetic keeps the pointer in the
  // shared window so the compiler emits LDS/STS rather than generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  EwChain* chain_s = reinterpret_cast<EwChain*>(smem + C::STAGES * C::STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int jid, tile;
  find_job(p.tile_start, p.njobs, blockIdx.x, jid, tile);
  const int tiles_n = p.tiles_n[jid];
  const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;

  int M, N, nstages;
  if constexpr (IS_DW) {
    M = p.job[jid].m;
    N = p.job[jid].n;
    nstages = (p.k + BK - 1) / BK;
  } else {
    M = p.rows;
    N = p.job[jid].n;
    nstages = 0;
    for (int s = 0; s < p.job[jid].nseg; ++s) nstages += (p.job[jid].seg[s].k + BK - 1) / BK;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], kProducers);  // every producer thread arrives after its own proxy fence
      mbar_init(&empty[s], 1);          // tcgen05.commit
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if constexpr (!IS_DW) {
    if (threadIdx.x < 256) stage_chain(chain_s, p.job[jid].epi, threadIdx.x, 256);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ---------------- producers ----------------
    TileLoad<BM, IS_DW> la;
    TileLoad<BN, IS_DW> lb;
    int seg = 0, k0 = 0;
    for (int it = 0; it < nstages; ++it) {
      const int s = it % C::STAGES;
      // issue this stage's global loads before waiting for the slot to drain
      if constexpr (IS_DW) {
        const auto& jb = p.job[jid];
        la.load(Src{jb.e, jb.m, M, p.k, false}, m0, k0, threadIdx.x);
        lb.load(Src{jb.y, jb.n, N, p.k, false}, n0, k0, threadIdx.x);
        k0 += BK;
      } else {
        const Seg& sg = p.job[jid].seg[seg];
        const bool va = (sg.k % 4 == 0) && (reinterpret_cast<uintptr_t>(sg.a) % 16 == 0);
        const bool vb = (sg.k % 4 == 0) && (reinterpret_cast<uintptr_t>(sg.b) % 16 == 0);
        la.load(Src{sg.a, sg.k, M, sg.k, va}, m0, k0, threadIdx.x);
        lb.load(Src{sg.b, sg.k, N, sg.k, vb}, n0, k0, threadIdx.x);
        k0 += BK;
        if (k0 >= sg.k) {
          k0 = 0;
          ++seg;
        }
      }
      mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
      uint8_t* base = smem + s * C::STAGE_BYTES;
      la.store(reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + C::A_BYTES), threadIdx.x);
      lb.store(reinterpret_cast<float*>(base + 2 * C::A_BYTES),
               reinterpret_cast<float*>(base + 2 * C::A_BYTES + C::B_BYTES), threadIdx.x);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&full[s]);
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer (warp 8) ----------------
    const int n_inst = (N - n0) >= BN ? BN : (((N - n0) + 15) / 16) * 16;
    const uint32_t idesc = idesc_tf32(BM, n_inst, 0, 0);  // both operands K-major in smem
    const bool split = p.terms != 1;
    for (int it = 0; it < nstages; ++it) {
      const int s = it % C::STAGES;
      mbar_wait(&full[s], (it / C::STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = smem_u32(smem + s * C::STAGE_BYTES);
      const uint32_t a_hi = base, a_lo = base + C::A_BYTES;
      const uint32_t b_hi = base + 2 * C::A_BYTES, b_lo = b_hi + C::B_BYTES;
#pragma unroll
      for (int j = 0; j < BK / 8; ++j) {
        // K-major SW128: the j-th 8-deep k-step starts 32 B into each swizzled
        // 128-byte row; 8-row groups are 1024 B apart (SBO); LBO unused.
        const uint32_t off = j * 32;
        const uint64_t dah = smem_desc(a_hi + off, 16, 1024), dal = smem_desc(a_lo + off, 16, 1024);
        const uint64_t dbh = smem_desc(b_hi + off, 16, 1024), dbl = smem_desc(b_lo + off, 16, 1024);
        const uint32_t acc0 = (it > 0 || j > 0) ? 1u : 0u;
        if (split) {
          mma_tf32(tmem, dal, dbh, idesc, acc0);  // small terms first
          mma_tf32(tmem, dah, dbl, idesc, 1u);
        }
        mma_tf32(tmem, dah, dbh, idesc, split ? 1u : acc0);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(done);
  }

  // ---------------- epilogue (warps 0-7) ----------------
  if (warp < 8) {
    mbar_wait(done, 0);
    if (threadIdx.x == 0) { TRACE(3, 0) }
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // all MMAs are complete: the pipeline smem is free for the staging tile
    epilogue<BN, IS_DW>(p, jid, m0, n0, M, N, tmem, reinterpret_cast<float*>(smem), chain_s, threadIdx.x, 0, 0, 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 8) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

// ---------------------------------------------------------------------------
// TMA-fed tensor-core GEMM (NT form with the elementwise-chain epilogue, and
// the dW form).  Warp roles: warp 8 lane 0 issues one TMA load per operand and
// stage (raw fp32; the tensor core truncates it to its tf32 "hi" part), the 8
// converter warps form x_lo = x - trunc(x) for both operands at the same byte
// offsets (the swizzle is position-independent), warp 9 lane 0 issues the
// three tcgen05.mma per 8-deep k-step.  Three mbarriers per stage: TMA landed
// -> residuals written -> MMAs done (tcgen05.commit frees the slot).
//
// PAIR = true runs a CTA pair (cluster of 2 on one TPC, tcgen05 cta_group::2):
// the pair computes a 256 x BN tile; each CTA loads and converts its own 128
// rows of A and HALF of B (BN/2 rows) and holds its 128 accumulator rows in its
// own TMEM, the leader (rank 0) issues M=256 MMAs that read both CTAs' shared
// memory.  Per CTA this halves the B bytes written by TMA, converted and read
// by the tensor core -- the kernel is shared-memory-bandwidth bound
// (tools/gemm_bench.py trace build: 288 KB of smem traffic per 32-deep stage at
// 128x256 vs 1536 MMA cycles).
constexpr int kTmaThreads = 352;  // warps 0-7 convert + epilogue, 8 and 10 TMA, 9 MMA

// TA: the A operand's tf32 hi/lo halves live in tensor memory (converter
// warps tcgen05.st them), so the tensor core reads only B from shared memory.
// Shared memory per stage: [A raw][B][B_lo] (TA) or [A][A_lo][B][B_lo].
template <int BN, int BNL, int BKT, bool TA>
struct TCfg {
  static constexpr int BK = BKT;
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BNL * BK * 4;  // this CTA's B rows
  static constexpr int B_OFF = TA ? A_BYTES : 2 * A_BYTES;
  static constexpr int STAGE_BYTES = B_OFF + 2 * B_BYTES;
  static constexpr int RAW = 196608 / STAGE_BYTES;
  static constexpr int TMEM_CAP = TA ? (512 - BN) / 64 : 8;  // A stages of 64 TMEM columns
  static constexpr int CAP = TMEM_CAP < 8 ? TMEM_CAP : 8;
  static constexpr int STAGES = RAW > CAP ? CAP : (RAW < 2 ? 2 : RAW);
  static constexpr int TMEM_COLS = TA ? 512 : (BN < 32 ? 32 : BN);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + kChainBytes;
  static_assert(BM * (BN + 4) * 4 <= STAGES * STAGE_BYTES, "epilogue staging must fit in the pipeline smem");
  static_assert(!TA || BK == 32, "TMEM A path reads the SWIZZLE_128B K-major layout");
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_tf32_ta_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                                 uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

template <int ROWS>
__host__ __device__ constexpr int box_idx() {  // 32/64/128/256-row map variant
  return ROWS == 32 ? 0 : (ROWS == 64 ? 1 : (ROWS == 128 ? 2 : 3));
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 16-byte load from the same shared-memory offset in cluster CTA `rank`
__device__ __forceinline__ float4 ld_dsmem4(const float* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote)
               : "memory");
  return v;
}

// arrive on the mbarrier at the same smem offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// wait with cluster-scope acquire (arrivals from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// commit to the mbarrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint32_t leader = 0) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)(3u << leader))
      : "memory");
}

template <int BN, bool IS_DW, bool PAIR, class P>
__global__ void __launch_bounds__(kTmaThreads, 1) tma_gemm_kernel(const __grid_constant__ P p) {
  constexpr int NCTA = PAIR ? 2 : 1;
  constexpr int BNL = BN / NCTA;  // B rows held by this CTA
#ifdef RGB_EXP_NO_TMEM_A
  constexpr bool TA = false;
#else
  constexpr bool TA = !IS_DW && kTmaNtBk == 32;
#endif
  using C = TCfg<BN, BNL, IS_DW ? 32 : kTmaNtBk, TA>;
  constexpr int BK = C::BK;
  constexpr int kBoxIdx = box_idx<BNL>();
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SWIZZLE_128B); offset arithmetic keeps the pointer in the
  // shared window so the compiler emits LDS/STS rather than generic LD/ST.
  // Both CTAs of a pair get the same layout (the leader's MMA descriptors
  // address the peer's operands at the same offsets).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // Plain TF32 (p.terms == 1, single CTAs): no residual halves, so the same
  // shared memory holds more logical stages of [A][B] (TA: 32 instead of 64
  // TMEM columns per A stage); the barrier arrays are sized for 8 stages.
  constexpr int kMaxSt = 8;
  static_assert(C::STAGES <= kMaxSt && 3 * kMaxSt * 8 + 12 <= 256, "barrier region");
  const bool one = !PAIR && p.terms == 1;
  const int SB = one ? C::A_BYTES + C::B_BYTES : C::STAGE_BYTES;
  const int BOFF = one ? C::A_BYTES : C::B_OFF;
  const int TST = one ? 32 : 64;  // TMEM columns per TA stage
  int NST = C::STAGES;
  if (one) {
    NST = (C::STAGES * C::STAGE_BYTES) / SB;
    if (TA && NST > (512 - BN) / 32) NST = (512 - BN) / 32;
    if (NST > kMaxSt) NST = kMaxSt;
  }
  uint64_t* tma_full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* conv_full = tma_full + kMaxSt;
  uint64_t* empty = conv_full + kMaxSt;
  uint64_t* done = empty + kMaxSt;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  EwChain* chain_s = reinterpret_cast<EwChain*>(smem + C::STAGES * C::STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster rank: a pair is ranks (2i, 2i+1) (cta_group::2 peers differ in
  // bit 0); with cluster split-K a pair tile's splits are pairs 0..splits-1
  const uint32_t ctarank = PAIR ? cluster_rank() : 0;
  const uint32_t rank = ctarank & 1u;        // rank inside the CTA pair
  const uint32_t leader = ctarank & ~1u;     // the pair's MMA-issuing CTA
  CTA_MARK(0)
  int jid, tile;
  // block -> (output tile, split, pair rank); the splits of one tile are adjacent
  const int blk = blockIdx.x / NCTA;
  int splits = 1, split = 0, tile_lin = blk, csplit = 1;
  if constexpr (!IS_DW) {
    splits = p.splits > 1 ? p.splits : 1;
    split = blk % splits;
    tile_lin = blk / splits;
    if (p.csplit) csplit = splits;  // splits reduced inside the cluster (no scratch)
  }
  find_job(p.tile_start, p.njobs, tile_lin, jid, tile);
  const auto& job = p.job[jid];
  const int tiles_n = p.tiles_n[jid];
  const int m0 = (tile / tiles_n) * (BM * NCTA) + (int)rank * BM;  // this CTA's accumulator rows
  const int n0 = (tile % tiles_n) * BN;
  const int nb0 = n0 + (int)rank * BNL;                             // this CTA's B rows
  int M, N, nstages;
  if constexpr (IS_DW) {
    M = job.m;
    N = job.n;
    nstages = (p.k + BK - 1) / BK;
  } else {
    M = p.rows;
    N = job.n;
    nstages = 0;
    for (int s = 0; s < job.nseg; ++s) nstages += (job.seg[s].k + BK - 1) / BK;
  }
  // this block's K-stage range [s_begin, s_begin + nstages)
  const int s_begin = (int)((long long)split * nstages / splits);
  nstages = (int)((long long)(split + 1) * nstages / splits) - s_begin;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&tma_full[s], 2);  // one expect_tx arrival per producer warp
      // pair: one arrival per converter warp of both CTAs (on the leader's copy)
      mbar_init(&conv_full[s], PAIR ? 2 : kProducers);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if constexpr (!IS_DW) {
    if (threadIdx.x < 256) stage_chain(chain_s, p.job[jid].epi, threadIdx.x, 256);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) {
    cluster_sync();  // peer barriers initialised before any remote arrive
  } else {
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // PDL (frame loops): only the A operand and the epilogue touch data the
  // predecessor kernel writes; the weight (B) loads and the whole SMEM/TMEM
  // pipeline start before it completes.  IS_DW launches are never PDL.
  pdl_trigger();

  if (warp == 8 || warp == 10) {
    if (lane == 0) {
      // ---------------- TMA producers: warp 8 loads A, warp 10 loads B ----------------
      // (two issuing warps: a single thread's TMA instructions complete one
      // after another at ~25-55 B/clk per SM -- tools/tma_probe.cu)
      const bool load_a = warp == 8;
      if (load_a) pdl_wait();
      int seg = 0, k0 = 0;
      if constexpr (!IS_DW) {
        for (int skip = s_begin; skip > 0;) {  // locate the first stage of this split
          const int ns = (job.seg[seg].k + BK - 1) / BK;
          if (skip >= ns) {
            skip -= ns;
            ++seg;
          } else {
            k0 = skip * BK;
            skip = 0;
          }
        }
      }
      for (int it = 0; it < nstages; ++it) {
        const int s = it % NST;
        mbar_wait(&empty[s], ((it / NST) & 1) ^ 1);
        if (load_a) { TRACE(0, it) }
        uint8_t* base = smem + s * SB;
        mbar_expect_tx(&tma_full[s], load_a ? C::A_BYTES : C::B_BYTES);
        if constexpr (IS_DW) {
          // MN-contiguous E [K x M] and Y [K x N]: one 3-D box of 4 (BNL/32)
          // 4-KB atoms {32 mn, 32 k} per operand (rgb_plan.cu encode_map_mn)
          if (load_a) tma_load_3d(base, map_at(job.te, 2), 0, job.erow + k0, m0 / 32, &tma_full[s]);
          else tma_load_3d(base + BOFF, map_at(job.ty, kBoxIdx), 0, job.yrow + k0, nb0 / 32, &tma_full[s]);
          k0 += BK;
        } else {
          const Seg& sg = job.seg[seg];
          if (load_a) tma_load_2d(base, sg.ta, k0, sg.arow + m0, &tma_full[s]);
          // weight maps come in 32/64/128/256-row box variants: one load per stage
          else tma_load_2d(base + BOFF, map_at(sg.tb, kBoxIdx), k0, nb0, &tma_full[s]);
          k0 += BK;
          if (k0 >= sg.k) {
            k0 = 0;
            ++seg;
          }
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (the leader of a pair) ----------------
      // pair: always the full BN (B rows past N are zero-filled by TMA, the
      // epilogue skips those columns) so that each CTA's half is BN/2 rows
      const int n_inst = (PAIR || (N - n0) >= BN) ? BN : (((N - n0) + 15) / 16) * 16;
      const uint32_t idesc = idesc_tf32(BM * NCTA, n_inst, IS_DW ? 1 : 0, IS_DW ? 1 : 0);
      const bool split = p.terms != 1;  // 3xTF32 lo terms (plain TF32 issues only hi*hi)
      for (int it = 0; it < nstages; ++it) {
        const int s = it % NST;
        if constexpr (PAIR) mbar_wait_cluster(&conv_full[s], (it / NST) & 1);
        else mbar_wait(&conv_full[s], (it / NST) & 1);
        TRACE(2, it)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = smem_u32(smem + s * SB);
        const uint32_t a_hi = base, a_lo = base + C::A_BYTES;
        const uint32_t b_hi = base + BOFF, b_lo = b_hi + C::B_BYTES;
        const uint32_t ta_hi = tmem + BN + TST * s, ta_lo = ta_hi + 32;  // TA: A stage in TMEM
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          uint64_t dah, dal, dbh, dbl;
          if constexpr (IS_DW) {
            // MN-major SWIZZLE_128B_BASE32B: 32-wide MN atoms 4 KB apart (LBO),
            // 4-row K groups 512 B apart (SBO); an 8-deep k-step is 1 KB
            const uint32_t off = j * 1024;
            dah = smem_desc(a_hi + off, 4096, 512, 1);
            dal = smem_desc(a_lo + off, 4096, 512, 1);
            dbh = smem_desc(b_hi + off, 4096, 512, 1);
            dbl = smem_desc(b_lo + off, 4096, 512, 1);
          } else {
            // K-major SWIZZLE_128B (BK 32: 128-byte rows, 8-row groups 1 KB
            // apart) or SWIZZLE_64B (BK 16: 64-byte rows, groups 512 B apart);
            // the j-th 8-deep k-step starts 32 B into each row
            constexpr uint32_t sbo = BK * 32, lay = BK == 32 ? 2 : 4;
            const uint32_t off = j * 32;
            dah = smem_desc(a_hi + off, 16, sbo, lay);
            dal = smem_desc(a_lo + off, 16, sbo, lay);
            dbh = smem_desc(b_hi + off, 16, sbo, lay);
            dbl = smem_desc(b_lo + off, 16, sbo, lay);
          }
          const uint32_t acc0 = (it > 0 || j > 0) ? 1u : 0u;
          if constexpr (TA) {
            // A hi/lo from tensor memory: 8 columns per k-step
            const uint32_t acch = split ? 1u : acc0;
            if constexpr (PAIR) {
              if (split) {
                mma_tf32_ta_pair(tmem, ta_lo + 8 * j, dbh, idesc, acc0);
                mma_tf32_ta_pair(tmem, ta_hi + 8 * j, dbl, idesc, 1u);
              }
              mma_tf32_ta_pair(tmem, ta_hi + 8 * j, dbh, idesc, acch);
            } else {
              if (split) {
                mma_tf32_ta(tmem, ta_lo + 8 * j, dbh, idesc, acc0);
                mma_tf32_ta(tmem, ta_hi + 8 * j, dbl, idesc, 1u);
              }
              mma_tf32_ta(tmem, ta_hi + 8 * j, dbh, idesc, acch);
            }
          } else if constexpr (PAIR) {
            if (split) {
              mma_tf32_pair(tmem, dal, dbh, idesc, acc0);
              mma_tf32_pair(tmem, dah, dbl, idesc, 1u);
            }
            mma_tf32_pair(tmem, dah, dbh, idesc, split ? 1u : acc0);
          } else {
            if (split) {
              mma_tf32(tmem, dal, dbh, idesc, acc0);
              mma_tf32(tmem, dah, dbl, idesc, 1u);
            }
            mma_tf32(tmem, dah, dbh, idesc, split ? 1u : acc0);
          }
        }
        if constexpr (PAIR) mma_commit_pair(&empty[s], leader);
        else mma_commit(&empty[s]);
      }
      if constexpr (PAIR) mma_commit_pair(done, leader);
      else mma_commit(done);
    }
  } else {
    // ---------------- converters: x_lo = x - trunc(x), same byte offsets ----------------
    for (int it = 0; it < nstages; ++it) {
      const int s = it % NST;
      mbar_wait(&tma_full[s], (it / NST) & 1);
      if (threadIdx.x == 0) { TRACE(1, it) }
      uint8_t* base = smem + s * SB;
#ifndef RGB_EXP_NOCONV
      if constexpr (TA) {
        // A row r = 32*(warp%4) + lane (the TMEM lane quarter this warp may
        // access), K half (warp/4): 16-B chunk c of row r sits at (c ^ (r%8))
        // in the SWIZZLE_128B layout; hi = raw (the MMA truncates), lo = residual
        const int quarter = warp & 3, kh = warp >> 2, r = quarter * 32 + lane;
        const uint8_t* arow = base + r * 128;
        float hi[16], lo[16];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c = kh * 4 + cc;
          const float4 x = *reinterpret_cast<const float4*>(arow + ((c ^ (r & 7)) * 16));
          hi[4 * cc] = x.x, hi[4 * cc + 1] = x.y, hi[4 * cc + 2] = x.z, hi[4 * cc + 3] = x.w;
        }
        if (p.terms != 1) {
#pragma unroll
          for (int q = 0; q < 16; ++q) lo[q] = tf32_residual(hi[q]);
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) hi[q] = tf32_rna(hi[q]);  // plain TF32: round, do not truncate
        }
        const uint32_t ta = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + BN + TST * s + 16 * kh;
        tmem_st16(ta, hi);
        if (p.terms != 1) tmem_st16(ta + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      } else if (p.terms != 1) {
        const float4* a_hi = reinterpret_cast<const float4*>(base);
        float4* a_lo = reinterpret_cast<float4*>(base + C::A_BYTES);
#pragma unroll
        for (int i = 0; i < C::A_BYTES / 16 / kProducers; ++i) {
          const int q = threadIdx.x + i * kProducers;
          const float4 x = a_hi[q];
          a_lo[q] = make_float4(tf32_residual(x.x), tf32_residual(x.y), tf32_residual(x.z), tf32_residual(x.w));
        }
      }
      if (p.terms != 1) {  // B residual (weights for the NT form, activations for dW)
        const float4* b_hi = reinterpret_cast<const float4*>(base + BOFF);
        float4* b_lo = reinterpret_cast<float4*>(base + BOFF + C::B_BYTES);
        for (int q = threadIdx.x; q < C::B_BYTES / 16; q += kProducers) {
          const float4 x = b_hi[q];
          b_lo[q] = make_float4(tf32_residual(x.x), tf32_residual(x.y), tf32_residual(x.z), tf32_residual(x.w));
        }
      } else {
        // plain TF32: round every smem operand to nearest (cvt.rna) in place --
        // the MMA alone would truncate (a 2^-11 relative bias on every product)
        if constexpr (!TA) round_tf32_inplace(base, C::A_BYTES, threadIdx.x, kProducers);
        round_tf32_inplace(base + BOFF, C::B_BYTES, threadIdx.x, kProducers);
      }
      if (threadIdx.x == 0) { TRACE(4, it) }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (threadIdx.x == 0) { TRACE(5, it) }
#endif
      if constexpr (PAIR) {
        // one arrival per CTA: a cluster-scope release costs a GPU-scope
        // MEMBAR (ncu: 20% of converter stall cycles when every warp arrived)
        asm volatile("bar.sync 2, 256;" ::: "memory");
        if (threadIdx.x == 0) {
          if (rank == 0) mbar_arrive(&conv_full[s]);
          else mbar_arrive_cluster(&conv_full[s], leader);
        }
      } else {
        mbar_arrive(&conv_full[s]);
      }
    }
    // ---------------- epilogue ----------------
    pdl_wait();  // the epilogue reads / writes global data of the frame
    mbar_wait(done, 0);
    if (threadIdx.x == 0) { TRACE(3, 0) }
    CTA_MARK(1)
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // split-K partial tiles are indexed by 128-row tile: pair tile * 2 + rank;
    // cluster split-K stops after staging the partial accumulator in smem
    epilogue<BN, IS_DW>(p, jid, m0, n0, M, N, tmem, reinterpret_cast<float*>(smem), chain_s, threadIdx.x,
                        tile_lin * NCTA + (int)rank, split, csplit > 1 ? 1 : splits, 0, BM, csplit > 1 ? 1 : 3);
    CTA_MARK(2)
  }
  if constexpr (!IS_DW) {
    if (csplit > 1) {
      // cluster split-K: the splits of this tile are one cluster; CTA `split`
      // sums rows [split*BM/csplit, ...) of all partial tiles in split order
      // through distributed shared memory and runs the epilogue on them (with
      // pairs: over the split CTAs of the same pair rank, cluster ranks 2k+rank)
      __syncwarp();
      cluster_sync();
      const int r_lo = split * BM / csplit, r_hi = (split + 1) * BM / csplit;
      float* tile_s = reinterpret_cast<float*>(smem);
      if (warp < 8) {
        // every remote load of a batch is in flight before the first is used
        // (a DSMEM round trip is ~200 cycles; the serial form cost ~1 us more
        // per frame, tools/trace_frame_loop.py)
        constexpr int G4 = BN / 4;
        using CE = Cfg<BN>;
        const int nq = (r_hi - r_lo) * G4;
        for (int q0 = threadIdx.x; q0 < nq; q0 += 256 * 4) {
          float4 a[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int q = q0 + 256 * i;
            a[i] = q < nq ? ld_dsmem4(tile_s + (r_lo + q / G4) * CE::EPI_LD + (q % G4) * 4, PAIR ? rank : 0u)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          for (int k = 1; k < csplit; ++k) {
            float4 b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int q = q0 + 256 * i;
              b[i] = q < nq ? ld_dsmem4(tile_s + (r_lo + q / G4) * CE::EPI_LD + (q % G4) * 4,
                                        PAIR ? (uint32_t)(2 * k) + rank : (uint32_t)k)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = add4(a[i], b[i]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int q = q0 + 256 * i;
            if (q < nq) *reinterpret_cast<float4*>(tile_s + (r_lo + q / G4) * CE::EPI_LD + (q % G4) * 4) = a[i];
          }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        CTA_MARK(3)
        epilogue<BN, IS_DW>(p, jid, m0, n0, M, N, tmem, tile_s, chain_s, threadIdx.x, 0, 0, 1, r_lo, r_hi, 2);
        CTA_MARK(4)
      }
      __syncwarp();
      cluster_sync();  // peers are done reading this CTA's partial tile
      CTA_MARK(5)
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) {
    cluster_sync();  // the pair's MMAs and remote arrivals are complete before teardown
  } else {
    __syncthreads();
  }
  if (warp == 9) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
    } else {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
    }
  }
}

template <int BN, bool IS_DW, class P>
void launch_one(P p, int tiles, cudaStream_t s) {
  static bool configured = false;
  auto k = tc_gemm_kernel<BN, IS_DW, P>;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
    configured = true;
  }
  k<<<tiles, kThreads, Cfg<BN>::SMEM, s>>>(p);
}

// blocks = CTAs (2 per pair tile when PAIR)
// ---------------------------------------------------------------------------
// Persistent form of the TMA kernel for launches of several waves: each CTA
// (pair) walks output tiles blockIdx, blockIdx + grid, ...; two chunk
// accumulators in TMEM let 8 dedicated epilogue warps fold / drain one while
// the producers, converters and MMA issuer fill the other (in the one-tile
// kernel the epilogue was ~25% of every multi-wave launch).
//   warps 0-3 converters, 4-11 epilogue (two groups), 12 TMA A, 13 MMA, 14 TMA B;
//   setmaxnreg moves registers from the converter / producer warp groups to
//   the epilogue, whose threads hold the tile's running sum (BN/2 floats).
// Barriers: per stage tma_full / conv_full / empty (as above), per chunk
// accumulator x_full (MMA commit -> epilogue) / x_empty (epilogue -> MMA).
// The epilogue stages 16-column chunks of the tile in a private smem slice
// (registers -> smem -> coalesced 16-byte row walk).
//
// K-chunked accumulation.  tcgen05 adds each k-step's products into the fp32
// TMEM accumulator with truncation (round toward zero) in the alignment, so
// one accumulator's relative error grows linearly with the number of MMAs it
// absorbs (tools/accum_probe.py: 3xTF32 at K = 16384 -> 1.2e-4 random /
// 3.1e-4 coherent data vs 6e-6 for SIMT fp32; the cfg4 dW depth h*S is
// 16384).  So for deep K the MMA issuer restarts a fresh chunk accumulator X
// every `kc` stages; the epilogue warps fold each finished chunk into the
// tile's running sum R -- held in the epilogue threads' registers -- with
// round-to-nearest fp32 adds (tcgen05.ld X -> FADD; R = X for chunk 0) and
// release X while the MMAs fill the other X; the output pass of tile i
// overlaps the MMAs of tile i+1.  Truncation then acts on <= 3*kc*(BK/8)
// accumulations per chunk.  (Round 2 first kept R in TMEM beside a single
// chunk accumulator at 256-column tiles, so the MMA waited for every fold:
// ~6% of the cfg4 step; R in registers with two X removes the wait.)
#ifndef RGB_PERS_BWD3
#define RGB_PERS_BWD3 1  // 1: product-layer chains through chain_bwd3 / chain_fwd2
#endif
#ifndef RGB_PERS_SPEC
// 1: the chain epilogue uses the specialised ops (every operand of an op
// loaded before its first store: one memory latency per op instead of two)
#define RGB_PERS_SPEC 1
#endif
#ifndef RGB_PERS_RE
#define RGB_PERS_RE 2  // rows per thread per pass of the persistent epilogue's row walk
#endif
constexpr int kPersThreads = 512;  // 4 warp groups: converters | epilogue 0 | epilogue 1 | TMA A, MMA, TMA B
constexpr int kPersConv = 128;    // converter threads (warps 0-3)
constexpr int kEpiCols = 16;    // columns per epilogue chunk
constexpr int kEpiLd = 20;      // padded chunk row (floats)

template <int BN, int BNL>
struct PCfg {
  static constexpr int BK = 32;
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BNL * BK * 4;
  static constexpr int B_OFF = 2 * A_BYTES;
  static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
  static constexpr int CHUNK_BYTES = 2 * BM * kEpiLd * 4;  // one staging chunk per epilogue group
  static constexpr int BUDGET = 227 * 1024 - 1024 - 512 - 2 * kChainBytes - CHUNK_BYTES;
  static constexpr int RAW = BUDGET / STAGE_BYTES;
  static constexpr int STAGES = RAW > 8 ? 8 : RAW;
  // TMEM: two chunk accumulators X (the running sum lives in the epilogue's registers)
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 512 + 2 * kChainBytes + CHUNK_BYTES;
  static_assert(STAGES >= 2, "persistent pipeline needs two stages");
  static_assert(TMEM_COLS <= 512, "two chunk accumulators fit TMEM");
};

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// tile geometry shared by every role of the persistent kernel
template <int BN, bool IS_DW, bool PAIR, class P>
struct PTile {
  int jid, m0, n0, nb0, M, N, nstages, width;
  // t >= tail: the last wave's tiles cut in two column halves (tail split),
  // half h of tile tail + h / 2
  __device__ __forceinline__ PTile(const P& p, int t, uint32_t rank, int tail) {
    constexpr int NCTA = PAIR ? 2 : 1;
    int tile, half = -1;
    if (t >= tail) {
      half = (t - tail) & 1;
      t = tail + (t - tail) / 2;
    }
    find_job(p.tile_start, p.njobs, t, jid, tile);
    const int tiles_n = p.tiles_n[jid];
    m0 = (tile / tiles_n) * (BM * NCTA) + (int)rank * BM;
    n0 = (tile % tiles_n) * BN;
    width = BN;
    if (half >= 0) {
      width = BN / 2;
      n0 += half * width;
    }
    nb0 = n0 + (int)rank * (width / NCTA);
    if constexpr (IS_DW) {
      M = p.job[jid].m;
      N = p.job[jid].n;
      nstages = (p.k + 31) / 32;
    } else {
      M = p.rows;
      N = p.job[jid].n;
      nstages = 0;
      for (int s = 0; s < p.job[jid].nseg; ++s) nstages += (p.job[jid].seg[s].k + 31) / 32;
    }
  }
};

// The forward chain of a gate feeding a product layer (the LSTM out_gate ->
// out_prod: engine.py:405-413 hoisted): op 0 g = act(acc + terms + rank-1),
// op 1 p = f_0 * f_1 with g one of the factors.  The other factor, the terms
// and the rank-1 operands are loaded up front and g is forwarded: one memory
// latency per row group instead of two.  Arithmetic exactly as ew_apply_vec.
__device__ __forceinline__ bool chain_is_fwd2(const EwChain& ch) {
  if (ch.nops != 2) return false;
  const EwOp &o = ch.op[0], &m = ch.op[1];
  if (o.kind != EW_FWD_ADD || o.base || o.nterm > 2 || o.nrank1 > 1) return false;
  if (m.kind != EW_FWD_MUL || m.nfac != 2 || (m.fac[0] != o.out) == (m.fac[1] != o.out)) return false;
  for (int i = 0; i < o.nterm; ++i)
    if (o.term[i] == o.out) return false;
  return m.out != o.out && m.out != m.fac[0] && m.out != m.fac[1];
}

template <int R>
__device__ __forceinline__ void chain_fwd2(const EwChain& ch, int width, const int64_t (&r)[R], int j,
                                           const bool (&ok)[R], const RingWrite& ring, const float4 (&acc)[R]) {
  const EwOp &o = ch.op[0], &m = ch.op[1];
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const int gi = m.fac[0] == o.out ? 0 : 1;
  int64_t e[R];
  float4 t0[R], t1[R], x[R];
  float src[R];
  const bool r1 = o.nrank1 > 0;
  const float4 w = r1 ? ld4(o.r1w[0], j) : zero;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    e[u] = r[u] * width + j;
    t0[u] = (o.nterm > 0 && ok[u]) ? ld4(o.term[0], e[u]) : zero;
    t1[u] = (o.nterm > 1 && ok[u]) ? ld4(o.term[1], e[u]) : zero;
    x[u] = ok[u] ? ld4(m.fac[1 - gi], e[u]) : zero;
    src[u] = (r1 && ok[u]) ? o.r1src[0][r[u]] : 0.0f;
  }
#pragma unroll
  for (int u = 0; u < R; ++u) {
    if (!ok[u]) continue;
    float4 v = acc[u];
    if (o.nterm > 0) v = add4(v, t0[u]);
    if (o.nterm > 1) v = add4(v, t1[u]);
    if (r1) v = add4(v, make_float4(w.x * src[u], w.y * src[u], w.z * src[u], w.w * src[u]));
    const float4 g = make_float4(act_apply(o.act, v.x), act_apply(o.act, v.y), act_apply(o.act, v.z),
                                 act_apply(o.act, v.w));
    ring_store4(o.out, e[u], r[u], width, o.out_is_ring, ring, g);
    ring_store4(m.out, e[u], r[u], width, m.out_is_ring, ring, gi == 0 ? mul4(g, x[u]) : mul4(x[u], g));
  }
}

// The backward chain of a product layer fed by a GEMM (the LSTM out_prod:
// engine.py:519-566): op 0 d = acc, eps_i = d * f_(1-i) over two co-factors;
// ops 1, 2 the two factor layers' deltas  d_q = (0 + eps_k) * f'(y_q).  Every
// operand the three ops read from memory (the co-factors, y_1, y_2) is loaded
// up front and the eps are forwarded in registers: one memory latency per row
// group instead of one per op.  Arithmetic exactly as ew_apply_vec.
__device__ __forceinline__ bool chain_is_bwd3(const EwChain& ch) {
  if (ch.nops != 3) return false;
  const EwOp& o = ch.op[0];
  if (o.kind != EW_BWD || o.act != ACT_IDENTITY || o.nterm || o.base || o.nrank1 || o.nfac != 2 || !o.eps[0] ||
      !o.eps[1] || o.inj || o.y)
    return false;
  for (int q = 1; q <= 2; ++q) {
    const EwOp& d = ch.op[q];
    if (d.kind != EW_BWD || (d.act != ACT_SIGMOID && d.act != ACT_TANH) || d.nterm != 1 || d.base || d.nrank1 ||
        d.nfac || d.inj || !d.y || (d.term[0] != o.eps[0] && d.term[0] != o.eps[1]))
      return false;
    // the deltas must not overwrite an operand a later op of the chain reads
    if (d.out == o.fac[0] || d.out == o.fac[1] || d.out == o.eps[0] || d.out == o.eps[1] || d.out == o.out) return false;
  }
  if (ch.op[1].out == ch.op[2].y || ch.op[2].out == ch.op[1].y || ch.op[1].out == ch.op[2].out) return false;
  return true;
}

__device__ __forceinline__ float4 bwd3_dact(int act, float4 y) {
  return make_float4(act_deriv(act, y.x), act_deriv(act, y.y), act_deriv(act, y.z), act_deriv(act, y.w));
}

template <int R>
__device__ __forceinline__ void chain_bwd3(const EwChain& ch, int width, const int64_t (&r)[R], int j,
                                           const bool (&ok)[R], const float4 (&acc)[R]) {
  const EwOp &o = ch.op[0], &p1 = ch.op[1], &p2 = ch.op[2];
  const float4 one = make_float4(1.f, 1.f, 1.f, 1.f), zero = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t e[R];
  float4 f0[R], f1[R], y1[R], y2[R];
#pragma unroll
  for (int u = 0; u < R; ++u) {
    e[u] = r[u] * width + j;
    f0[u] = ok[u] ? ld4(o.fac[0], e[u]) : one;
    f1[u] = ok[u] ? ld4(o.fac[1], e[u]) : one;
    y1[u] = ok[u] ? ld4(p1.y, e[u]) : zero;
    y2[u] = ok[u] ? ld4(p2.y, e[u]) : zero;
  }
#pragma unroll
  for (int u = 0; u < R; ++u) {
    if (!ok[u]) continue;
    const float4 d = acc[u];
    const float4 e0 = mul4(d, f1[u]), e1 = mul4(d, f0[u]);
    st4(o.out, e[u], d);
    st4(o.eps[0], e[u], e0);
    st4(o.eps[1], e[u], e1);
    const float4 t1 = p1.term[0] == o.eps[0] ? e0 : e1;
    const float4 t2 = p2.term[0] == o.eps[0] ? e0 : e1;
    st4(p1.out, e[u], mul4(add4(zero, t1), bwd3_dact(p1.act, y1[u])));
    st4(p2.out, e[u], mul4(add4(zero, t2), bwd3_dact(p2.act, y2[u])));
  }
}

template <int BN, bool IS_DW, bool PAIR, class P>
__global__ void __launch_bounds__(kPersThreads, 1) tma_gemm_persistent(const __grid_constant__ P p, int ntiles, int kc, int tail) {
  constexpr int NCTA = PAIR ? 2 : 1;
  constexpr int BNL = BN / NCTA;
  using C = PCfg<BN, BNL>;
  constexpr int BK = C::BK;
  constexpr int kBoxIdx = box_idx<BNL>();
  constexpr int HALF = BN / 2;  // running-sum columns per epilogue thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // Plain TF32 (p.terms == 1, single CTAs) needs no residual halves: each
  // physical [A][A_lo][B][B_lo] slot holds two logical [A][B] stages, so the
  // pipeline is twice as deep (2 -> 4 stages at BN = 256).
  const bool one = !PAIR && p.terms == 1;
  const int NST = one ? 2 * C::STAGES : C::STAGES;
  const int SB = one ? C::STAGE_BYTES / 2 : C::STAGE_BYTES;
  const int BOFF = one ? C::A_BYTES : C::B_OFF;
  if (kc <= 0) kc = 1 << 30;  // one chunk per tile
  static_assert(6 * C::STAGES * 8 + 4 * 8 + 8 <= 512, "barrier region");
  uint64_t* tma_full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* conv_full = tma_full + 2 * C::STAGES;
  uint64_t* empty = conv_full + 2 * C::STAGES;
  uint64_t* x_full = empty + 2 * C::STAGES;  // [2] chunk accumulators
  uint64_t* x_empty = x_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_empty + 2);
  EwChain* chain_s = reinterpret_cast<EwChain*>(smem + C::STAGES * C::STAGE_BYTES + 512);
  float* chunk_s = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 512 + 2 * kChainBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  const int first = blockIdx.x / NCTA, stride = gridDim.x / NCTA;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&tma_full[s], 2);
      mbar_init(&conv_full[s], PAIR ? 2 : kPersConv);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&x_full[b], 1);
      mbar_init(&x_empty[b], 2 * NCTA);  // both epilogue groups of every CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 13) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp >= 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;");
    if (warp == 12 || warp == 14) {
      if (lane == 0) {
        // ---------------- TMA producers (A: warp 12, B: warp 14) ----------------
        const bool load_a = warp == 12;
        int g = 0;  // global stage counter
        for (int t = first; t < ntiles; t += stride) {
          const PTile<BN, IS_DW, PAIR, P> T(p, t, rank, tail);
          const auto& job = p.job[T.jid];
          int seg = 0, k0 = 0;
          for (int it = 0; it < T.nstages; ++it, ++g) {
            const int s = g % NST;
            mbar_wait(&empty[s], ((g / NST) & 1) ^ 1);
            uint8_t* base = smem + s * SB;
            mbar_expect_tx(&tma_full[s], load_a ? C::A_BYTES : C::B_BYTES);
            if constexpr (IS_DW) {
              if (load_a) tma_load_3d(base, map_at(job.te, 2), 0, job.erow + k0, T.m0 / 32, &tma_full[s]);
              else tma_load_3d(base + BOFF, map_at(job.ty, kBoxIdx), 0, job.yrow + k0, T.nb0 / 32, &tma_full[s]);
              k0 += BK;
            } else {
              const Seg& sg = job.seg[seg];
              if (load_a) tma_load_2d(base, sg.ta, k0, sg.arow + T.m0, &tma_full[s]);
              else tma_load_2d(base + BOFF, map_at(sg.tb, kBoxIdx), k0, T.nb0, &tma_full[s]);
              k0 += BK;
              if (k0 >= sg.k) {
                k0 = 0;
                ++seg;
              }
            }
          }
        }
      }
    } else if (warp == 13 && lane == 0 && rank == 0) {
      // ---------------- MMA issuer: every chunk into a fresh X ----------------
      const uint32_t idesc_full = idesc_tf32(BM * NCTA, BN, IS_DW ? 1 : 0, IS_DW ? 1 : 0);
      const uint32_t idesc_half = idesc_tf32(BM * NCTA, BN / 2, IS_DW ? 1 : 0, IS_DW ? 1 : 0);
      const bool split = p.terms != 1;
      int g = 0, xc = 0;
      for (int t = first; t < ntiles; t += stride) {
        const PTile<BN, IS_DW, PAIR, P> T(p, t, rank, tail);
        int xb = -1, chunk_end = 0;
        uint32_t acc = tmem;
        const uint32_t idesc = T.width == BN ? idesc_full : idesc_half;
        for (int it = 0; it < T.nstages; ++it, ++g) {
          if (it == chunk_end) {  // next chunk: the other accumulator, once the epilogue folded it
            if (xb >= 0) {
              if constexpr (PAIR) mma_commit_pair(&x_full[xb]);
              else mma_commit(&x_full[xb]);
              ++xc;
            }
            xb = xc & 1;
            if constexpr (PAIR) mbar_wait_cluster(&x_empty[xb], ((xc >> 1) & 1) ^ 1);
            else mbar_wait(&x_empty[xb], ((xc >> 1) & 1) ^ 1);
            acc = tmem + xb * BN;
            chunk_end += kc;
          }
          const int s = g % NST;
          if constexpr (PAIR) mbar_wait_cluster(&conv_full[s], (g / NST) & 1);
          else mbar_wait(&conv_full[s], (g / NST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t base = smem_u32(smem + s * SB);
          const uint32_t a_hi = base, a_lo = base + C::A_BYTES;
          const uint32_t b_hi = base + BOFF, b_lo = b_hi + C::B_BYTES;
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {
            uint64_t dah, dal, dbh, dbl;
            if constexpr (IS_DW) {
              const uint32_t off = j * 1024;
              dah = smem_desc(a_hi + off, 4096, 512, 1);
              dal = smem_desc(a_lo + off, 4096, 512, 1);
              dbh = smem_desc(b_hi + off, 4096, 512, 1);
              dbl = smem_desc(b_lo + off, 4096, 512, 1);
            } else {
              const uint32_t off = j * 32;
              dah = smem_desc(a_hi + off, 16, 1024, 2);
              dal = smem_desc(a_lo + off, 16, 1024, 2);
              dbh = smem_desc(b_hi + off, 16, 1024, 2);
              dbl = smem_desc(b_lo + off, 16, 1024, 2);
            }
            const uint32_t acc0 = (it > chunk_end - kc || j > 0) ? 1u : 0u;
            if constexpr (PAIR) {
              if (split) {
                mma_tf32_pair(acc, dal, dbh, idesc, acc0);
                mma_tf32_pair(acc, dah, dbl, idesc, 1u);
              }
              mma_tf32_pair(acc, dah, dbh, idesc, split ? 1u : acc0);
            } else {
              if (split) {
                mma_tf32(acc, dal, dbh, idesc, acc0);
                mma_tf32(acc, dah, dbl, idesc, 1u);
              }
              mma_tf32(acc, dah, dbh, idesc, split ? 1u : acc0);
            }
          }
          if constexpr (PAIR) mma_commit_pair(&empty[s]);
          else mma_commit(&empty[s]);
        }
        if constexpr (PAIR) mma_commit_pair(&x_full[xb]);  // the tile's last chunk
        else mma_commit(&x_full[xb]);
        ++xc;
      }
    }
  } else if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    // ---------------- converters (warps 0-3) ----------------
    int g = 0;
    for (int t = first; t < ntiles; t += stride) {
      const PTile<BN, IS_DW, PAIR, P> T(p, t, rank, tail);
      for (int it = 0; it < T.nstages; ++it, ++g) {
        const int s = g % NST;
        mbar_wait(&tma_full[s], (g / NST) & 1);
        uint8_t* base = smem + s * SB;
        if (p.terms != 1) {
          const float4* a_hi = reinterpret_cast<const float4*>(base);
          float4* a_lo = reinterpret_cast<float4*>(base + C::A_BYTES);
#pragma unroll
          for (int i = 0; i < C::A_BYTES / 16 / kPersConv; ++i) {
            const int q = threadIdx.x + i * kPersConv;
            const float4 x = a_hi[q];
            a_lo[q] = make_float4(tf32_residual(x.x), tf32_residual(x.y), tf32_residual(x.z), tf32_residual(x.w));
          }
          const float4* b_hi = reinterpret_cast<const float4*>(base + BOFF);
          float4* b_lo = reinterpret_cast<float4*>(base + BOFF + C::B_BYTES);
#pragma unroll
          for (int i = 0; i < C::B_BYTES / 16 / kPersConv; ++i) {
            const int q = threadIdx.x + i * kPersConv;
            const float4 x = b_hi[q];
            b_lo[q] = make_float4(tf32_residual(x.x), tf32_residual(x.y), tf32_residual(x.z), tf32_residual(x.w));
          }
        } else {  // plain TF32: round both operands to nearest in place (the MMA would truncate)
          round_tf32_inplace(base, C::A_BYTES, threadIdx.x, kPersConv);
          round_tf32_inplace(base + BOFF, C::B_BYTES, threadIdx.x, kPersConv);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if constexpr (PAIR) {
          asm volatile("bar.sync 2, 128;" ::: "memory");
          if (threadIdx.x == 0) {
            if (rank == 0) mbar_arrive(&conv_full[s]);
            else mbar_arrive_cluster(&conv_full[s], 0);
          }
        } else {
          mbar_arrive(&conv_full[s]);
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ---------------- epilogue: two warp groups (4-7, 8-11) ----------------
    // Thread (lane quarter q, lane l) of group g owns accumulator row 32q+l,
    // columns {16-column chunks g, g+2, ...}: the tile's running sum R lives in
    // its registers.  Each finished chunk accumulator X is read (tcgen05.ld)
    // and added to R with round-to-nearest fp32 adds, then released to the MMA
    // -- which meanwhile fills the other X -- so the K-chunking costs no MMA
    // stall.  After the last chunk R goes through the group's SMEM staging
    // chunk to the coalesced output walk (chain epilogue or dW store).
    const int grp = warp >= 8 ? 1 : 0;
    const int et = threadIdx.x - (grp ? 8 : 4) * 32;  // 0..127
    const int quarter = warp & 3;                     // TMEM lane quarter this warp may read
    const int r_loc = quarter * 32 + lane;
    EwChain* my_chain = reinterpret_cast<EwChain*>(reinterpret_cast<uint8_t*>(chain_s) + grp * kChainBytes);
    float* my_chunk = chunk_s + grp * (BM * kEpiLd);
    const int bar = 3 + grp;
    auto gsync = [&] { asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory"); };
    float R[HALF];
    int staged_job = -1, xc = 0;
    bool bwd3 = false;  // the staged chain is the product-layer backward chain (chain_bwd3)
    bool fwd2 = false;  // ... the gate -> product forward chain (chain_fwd2)
    for (int t = first; t < ntiles; t += stride) {
      const PTile<BN, IS_DW, PAIR, P> T(p, t, rank, tail);
      const int nch = (T.nstages + kc - 1) / kc;
      for (int c = 0; c < nch; ++c, ++xc) {
        const int xb = xc & 1;
        mbar_wait(&x_full[xb], (xc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t xacc = tmem + xb * BN + (static_cast<uint32_t>(quarter * 32) << 16);
        // (a tail half tile folds stale columns into R too: never read)
#pragma unroll
        for (int q = 0; q < HALF / 16; ++q) {
          float v[16];
          tmem_ld16(xacc + grp * kEpiCols + q * 2 * kEpiCols, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) R[q * 16 + i] = c > 0 ? R[q * 16 + i] + v[i] : v[i];
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        gsync();
        if (et == 0) {
          if (rank == 0) mbar_arrive(&x_empty[xb]);
          else mbar_arrive_cluster(&x_empty[xb], 0);
        }
      }
      if constexpr (!IS_DW) {
        if (T.jid != staged_job) {  // the chain of this tile's job
          stage_chain(my_chain, p.job[T.jid].epi, et, 128);
          gsync();
          staged_job = T.jid;
          bwd3 = RGB_PERS_BWD3 && chain_is_bwd3(*my_chain);
          fwd2 = RGB_PERS_BWD3 && chain_is_fwd2(*my_chain);
        }
      }
      const int ncols = (T.N - T.n0) < T.width ? (T.N - T.n0) : T.width;
      const int nrows = (T.M - T.m0) < BM ? (T.M - T.m0) : BM;
      bool vec;
      float* g_out = nullptr;
      if constexpr (IS_DW) {
        g_out = p.job[T.jid].g;
        vec = T.N % 4 == 0 && aligned16(g_out);
      } else {
        vec = chain_vec_ok(*my_chain, T.N);
      }
#pragma unroll 1
      for (int q = 0; q < HALF / 16; ++q) {
        const int c0 = grp * kEpiCols + q * 2 * kEpiCols;
        if (c0 >= ncols) break;
        // this thread's 16 values of chunk q (selected without dynamic register indexing)
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = R[i];
#pragma unroll
        for (int qq = 1; qq < HALF / 16; ++qq)
          if (qq == q) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = R[qq * 16 + i];
          }
        float4* dst = reinterpret_cast<float4*>(my_chunk + r_loc * kEpiLd);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        gsync();
        const int cw = (ncols - c0) < kEpiCols ? (ncols - c0) : kEpiCols;
        if (vec) {
          // 4 lanes per row (16-byte groups), 32 rows per pass, RE rows per thread
          constexpr int RE = RGB_PERS_RE;
          const int sub = et >> 2, lc = et & 3, cl = lc * 4;
          if (cl < cw) {
#pragma unroll 1
            for (int rb = sub; rb < nrows; rb += 32 * RE) {
              int64_t rr[RE];
              bool ok[RE];
              float4 a4[RE];
#pragma unroll
              for (int u = 0; u < RE; ++u) {
                const int rl = rb + 32 * u;
                ok[u] = rl < nrows;
                rr[u] = T.m0 + (ok[u] ? rl : 0);
                a4[u] = *reinterpret_cast<const float4*>(my_chunk + (ok[u] ? rl : 0) * kEpiLd + cl);
              }
              if constexpr (IS_DW) {
#pragma unroll
                for (int u = 0; u < RE; ++u)
                  if (ok[u])
                    st4(g_out, rr[u] * T.N + T.n0 + c0 + cl,
                        make_float4(p.alpha * a4[u].x, p.alpha * a4[u].y, p.alpha * a4[u].z, p.alpha * a4[u].w));
              } else {
                const RingWrite ring = p.ring;
                if (bwd3) chain_bwd3<RE>(*my_chain, T.N, rr, T.n0 + c0 + cl, ok, a4);
                else if (fwd2) chain_fwd2<RE>(*my_chain, T.N, rr, T.n0 + c0 + cl, ok, ring, a4);
                else ew_chain_vec<RE, RGB_PERS_SPEC != 0>(*my_chain, T.N, rr, T.n0 + c0 + cl, ok, ring, true, a4);
              }
            }
          }
        } else {
          for (int e = et; e < nrows * cw; e += 128) {
            const int rl = e / cw, cl = e - rl * cw;
            const float a = my_chunk[rl * kEpiLd + cl];
            const int64_t r = T.m0 + rl;
            const int c = T.n0 + c0 + cl;
            if constexpr (IS_DW) {
              p.job[T.jid].g[r * T.N + c] = p.alpha * a;
            } else {
              const RingWrite ring = p.ring;
              for (int k = 0; k < my_chain->nops; ++k) ew_apply(my_chain->op[k], T.N, r, c, ring, k == 0, a);
            }
          }
        }
        gsync();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) cluster_sync();
  else __syncthreads();
  if (warp == 13) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
    } else {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
    }
  }
}

// ntiles output tiles (pair tiles when PAIR) over min(ntiles, SMs/NCTA) CTAs / pairs
// Truncating tensor-core accumulation (see tma_gemm_persistent): an
// accumulator absorbing more than this many K-stages (3 * 4 MMAs each in
// 3xTF32) loses ~1e-5 of its magnitude (a K = 1024 GEMM on coherent data
// measured 2.3e-5, tools/accum_probe.py) -- the end-to-end budget after
// several training steps is 1e-4 (tests/test_gpu_configs.py), so deeper
// launches run K-chunked.
constexpr int kMaxStagesPerAcc = 16;

// stages per accumulation chunk for a launch whose tiles are at most
// `max_stages` deep: 0 (one chunk per tile) when the whole K fits the bound,
// else 4 / 16 (3xTF32 dW / NT) or 12 / 48 (TF32) -- <= 48 / 192 truncating
// accumulations per chunk.
// RGB_TC_KC overrides (experiments).
int chunk_stages(int terms, int max_stages, bool dw) {
  static int forced = -1, forced_nt = -1;
  if (forced < 0) {
    const char* e = getenv("RGB_TC_KC");
    forced = e ? atoi(e) : 0;
    e = getenv("RGB_TC_KC_NT");
    forced_nt = e ? atoi(e) : 0;
  }
  const int per_acc = terms == 1 ? (max_stages + 2) / 3 : max_stages;
  if (per_acc <= kMaxStagesPerAcc) return 0;
  if (!dw && forced_nt > 0) return forced_nt;
  if (forced > 0) return forced;
  // dW (K = h*S, 16384 at cfg4): 4 stages per chunk (the folds cost the dW
  // epilogue nothing it cannot hide); the NT GEMMs (K <= 4096, chain-heavy
  // epilogues that are the kernel's bound): 16.  cfg4 after 5 training steps
  // (tools/diag_parity.py, profiles/r02_chunk_size_sweep.log): worst 4.9e-5;
  // NT 8 -> 4.3e-5 at -3% throughput, NT unchunked -> 8.8e-5 (too close to 1e-4)
  if (terms == 1) return dw ? 12 : 48;
  return dw ? 4 : 16;
}

template <int BN, bool IS_DW, bool PAIR, class P>
void launch_persistent(const P& p, int ntiles, int max_stages, cudaStream_t s) {
  using C = PCfg<BN, BN / (PAIR ? 2 : 1)>;
  static bool configured = false;
  auto k = tma_gemm_persistent<BN, IS_DW, PAIR, P>;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    configured = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int units = PAIR ? sms / 2 : sms;
  // tail split: when the last wave would hold at most half the units, its
  // tiles run as column halves on twice as many units (one half-length wave
  // instead of a full one; RGB_TC_TAIL=0 disables)
  static int tail_env = -1;
  if (tail_env < 0) {
    const char* e = getenv("RGB_TC_TAIL");
    tail_env = e ? atoi(e) != 0 : 1;
  }
  int tail = ntiles;
  const int rem = ntiles % units;
  if (!IS_DW && tail_env && ntiles > units && rem && 2 * rem <= units) {
    tail = ntiles - rem;
    ntiles += rem;
  }
  const int blocks = (ntiles < units ? ntiles : units) * (PAIR ? 2 : 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kPersThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = PAIR ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, p, ntiles, chunk_stages(p.terms, max_stages, IS_DW), tail);
}

template <int BN, bool IS_DW, bool PAIR, class P>
void launch_tma(const P& p, int blocks, cudaStream_t s, int cluster = 1) {
#ifdef RGB_EXP_NO_TMEM_A
  constexpr bool TA = false;
#else
  constexpr bool TA = !IS_DW && kTmaNtBk == 32;
#endif
  using C = TCfg<BN, BN / (PAIR ? 2 : 1), IS_DW ? 32 : kTmaNtBk, TA>;
  static bool configured = false;
  auto k = tma_gemm_kernel<BN, IS_DW, PAIR, P>;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    configured = true;
  }
  if (PAIR || cluster > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kTmaThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 * cluster : cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_active() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, k, p);
  } else if (pdl_active()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kTmaThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, p);
  } else {
    k<<<blocks, kTmaThreads, C::SMEM, s>>>(p);
  }
}

// 128-row tile index of output row r, tile column tn (pair launches number
// their 256-row tiles; each CTA of the pair owns tile * 2 + rank)
__device__ __forceinline__ int cta_tile(bool pair, int t0, int tiles_n, int64_t r, int tn) {
  if (!pair) return t0 + (int)(r / BM) * tiles_n + tn;
  return (t0 + (int)(r / (2 * BM)) * tiles_n + tn) * 2 + (int)((r / BM) & 1);
}

// Split-K fixup + epilogue: acc = sum of the partial tiles in split order,
// then the job's chain; one thread per 4 consecutive units of a row
// (blockIdx.y = job).
template <int BN>
__global__ void __launch_bounds__(256) splitk_epilogue_kernel(const __grid_constant__ GemmGroup p) {
  __shared__ __align__(16) int chain_words[sizeof(EwChain) / 4];
  const int j = blockIdx.y;
  stage_chain(reinterpret_cast<EwChain*>(chain_words), p.job[j].epi, threadIdx.x, blockDim.x);
  __syncthreads();
  const EwChain& ch = *reinterpret_cast<const EwChain*>(chain_words);
  const int N = p.job[j].n, M = p.rows, splits = p.splits, tiles_n = p.tiles_n[j], t0 = p.tile_start[j];
  const RingWrite ring = p.ring;
  const size_t tile_floats = (size_t)BM * BN;
  if (chain_vec_ok(ch, N)) {
    const int64_t nq = (int64_t)M * (N / 4);
    if (nq >= (int64_t)UINT32_MAX) __trap();
    const uint32_t w4 = (uint32_t)(N / 4);
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < (uint32_t)nq; q += gridDim.x * blockDim.x) {
      const uint32_t r32 = q / w4;
      const int64_t r = r32;
      const int c = (int)(q - r32 * w4) * 4;
      const int tl = cta_tile(p.pair != 0, t0, tiles_n, r, c / BN);
      const float* src = p.part + (size_t)tl * splits * tile_floats + (r % BM) * BN + (c % BN);
      float4 a = __ldcg(reinterpret_cast<const float4*>(src));
      for (int sp = 1; sp < splits; ++sp) a = add4(a, __ldcg(reinterpret_cast<const float4*>(src + sp * tile_floats)));
      const int64_t rr[1] = {r};
      const bool ok[1] = {true};
      const float4 acc[1] = {a};
      ew_chain_vec<1>(ch, N, rr, c, ok, ring, true, acc);
    }
  } else {
    const int64_t ne = (int64_t)M * N;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = e / N;
      const int c = (int)(e - r * N);
      const int tl = cta_tile(p.pair != 0, t0, tiles_n, r, c / BN);
      const float* src = p.part + (size_t)tl * splits * tile_floats + (r % BM) * BN + (c % BN);
      float a = __ldcg(src);
      for (int sp = 1; sp < splits; ++sp) a += __ldcg(src + sp * tile_floats);
      for (int k = 0; k < ch.nops; ++k) ew_apply(ch.op[k], N, r, c, ring, k == 0, a);
    }
  }
}


// ---------------------------------------------------------------------------
// Persistent frame loop of a recurrent SCC at large S.  The reference walks
// the frames of a recurrent supernode one at a time (engine.py:405-413
// forward, :568-576 backward); the per-frame work here is one grouped NT GEMM
// (the intra-SCC dense edges, e.g. cell(t-1) -> {in, forget} gates of an
// LSTM, [S x 1024] x [1024 x 2048] at cfg4) with the fused chain epilogue,
// optionally followed by elementwise steps (the LSTM cell update).  Launched
// once per frame that costs a launch, the TMEM / barrier prologue, a cold
// pipeline and the teardown per frame (~33 us per frame-step at cfg4 with a
// ~6 us tensor floor).  This kernel runs the whole loop:
//   * one cooperative launch (all CTAs co-resident; cluster split-K as in the
//     per-frame kernel), every CTA owns the same output tile (and K split) in
//     every frame; TMEM, barriers and the pipeline live across frames;
//   * the weight operand (B) does not depend on the frame: its TMA loads for
//     frame f+1 stream into free pipeline slots while frame f's epilogue and
//     the frame barrier run; only the state operand (A) waits for the barrier;
//   * frame f+1 starts after a grid barrier on frame f's outputs (release:
//     __threadfence + atomic; acquire + fence.proxy.async before the TMA
//     loads of A, which read what other SMs stored);
//   * split-K partial tiles are reduced through DSMEM with mbarrier handshakes
//     among the epilogue warps (part_ready / read_done), so the producer and
//     MMA warps never join a per-frame cluster barrier;
//   * the trailing elementwise steps of a frame run on all CTAs between two
//     grid barriers.
// Per-frame operands (segment rows, epilogue / elementwise pointers, ring
// mirror split) come from a device array of per-frame GemmGroup / EwLaunch
// blocks built once per (loop, ring phase) by the executor.
struct FrameLoop {
  const GemmGroup* frames;  // [nframes], loop order
  const EwLaunch* ew;       // [nframes * n_ew] or null
  int nframes, n_ew;
  int fuse_ew;              // 1: the elementwise steps run in the epilogue (element-local to the tile)
  int bu;                   // units per job in a tile (the tile's BN = njobs * bu)
  int prefetch;             // 1: warp 11 prefetches the chains' operands into L2 (off by default)
  int forward;              // 1: fused chain evaluation with register forwarding (frame_chains_fused)
  int pattern;              // 1 / 2: the LSTM cell forward / backward chains (lstm_chains), 0: generic
  int preload;              // 1: the pattern's operands are loaded before the split-K reduction (lstm_pre)
  const EwLaunch* tail;     // [nframes] or null: the one-op elementwise step after the loop, run in pass 1
  unsigned* bar;            // counter barrier: [0] arrivals (monotonic), [1] count at launch, [2] finished CTAs
};

template <int BN>
struct FCfg {
  static constexpr int BK = 32;
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;  // [A raw][B][B_lo] (A hi/lo go to TMEM)
  static constexpr int EPI_LD = BN + 4;
  static constexpr int TILE_BYTES = BM * EPI_LD * 4;         // dedicated epilogue staging tile
  static constexpr int CHAINS = 4;                           // chain slots (jobs, fused elementwise chains)
  static constexpr int BUDGET = 232448 - 1024 - 512 - CHAINS * kChainBytes - TILE_BYTES;
  static constexpr int RAW = BUDGET / STAGE_BYTES;
  static constexpr int TCAP = (512 - BN) / 64;               // A stages of 64 TMEM columns
  static constexpr int STAGES = RAW < TCAP ? (RAW > 8 ? 8 : RAW) : (TCAP > 8 ? 8 : TCAP);
  static constexpr int SMEM = STAGES * STAGE_BYTES + TILE_BYTES + 1024 + 512 + CHAINS * kChainBytes;
  static_assert(STAGES >= 2, "frame loop pipeline");
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Counter barrier of the frame loop (replaces a last-arriver generation flip:
// 1-1.5 instead of 2.5-3 us per forward frame, r02_frame_loop_counter_barrier.log).
// Waiters poll with relaxed loads and a short sleep (an acquire load per poll
// invalidates the SM's L1 -- measured to slow the epilogue warps' operand
// loads ~2x while the TMA / prefetch warps wait) and acquire once at the end.
// bar[0] counts arrivals monotonically
// across launches, bar[1] holds the count at the start of the running
// launch (written by the last CTA to finish the previous one, bar[2] counts
// finished CTAs).  Arrive = fence + fire-and-forget add (no last-arriver
// round trips: the waiters watch the counter itself); barrier k of a launch
// is complete when bar[0] >= base + k * nblocks.
__device__ __forceinline__ void ctr_arrive(unsigned* bar) {
  __threadfence();  // this CTA's stores before its arrival (cumulative over the bar.sync before it)
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}

__device__ __forceinline__ void ctr_wait(const unsigned* bar, unsigned target) {
  long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while ((int)(ld_relaxed_u32(bar) - target) < 0) {
    __nanosleep(32);
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000LL) __trap();  // 4 s: a lost CTA -- fail loudly instead of hanging the GPU
  }
  (void)ld_acquire_u32(bar);
}

// end of a launch: the last CTA publishes the arrival count as the next base
__device__ __forceinline__ void ctr_finish(unsigned* bar, unsigned next_base, unsigned nblocks) {
  __threadfence();
  if (atomicAdd(&bar[2], 1u) == nblocks - 1) {
    bar[2] = 0u;
    bar[1] = next_base;
    __threadfence();
  }
}

#ifdef RGB_FL_TRACE
__device__ long long g_fl_trace[64][16];  // CTA 0: per frame, globaltimer at the phase boundaries
__device__ int g_fl_frame;
__device__ __forceinline__ void fl_mark(int f, int e) {  // SM cycles (globaltimer ticks ~1 us)
  if (blockIdx.x == 0 && f < 64) g_fl_trace[f][e] = clock64();
}
#define FL_MARK(f, e) fl_mark(f, e)
#else
#define FL_MARK(f, e)
#endif

// ---- fused chain evaluation with register forwarding (frame loops) ----
// The ops of a frame's chains (every job's chain, then the fused elementwise
// steps) run back to back per element group in one thread.  An op's operand
// that an earlier op of the same group produced (same pointer: same buffer,
// frame and shift) is served from a 4-slot register cache instead of a
// store -> load round trip through global memory (~1 us each, measured with
// tools/trace_frame_loop.py); every other operand of every op is prefetched
// into L1 before the first op, so the group pays one memory latency instead
// of one per op.  Arithmetic per element is exactly ew_apply's.
template <int R>
struct FlCache {
  const float* p[4];
  float4 v[4][R];
};

template <int R>
__device__ __forceinline__ void fl_push(FlCache<R>& c, const float* p, const float4 (&v)[R]) {
#pragma unroll
  for (int sl = 3; sl > 0; --sl) {
    c.p[sl] = c.p[sl - 1];
#pragma unroll
    for (int u = 0; u < R; ++u) c.v[sl][u] = c.v[sl - 1][u];
  }
  c.p[0] = p;
#pragma unroll
  for (int u = 0; u < R; ++u) c.v[0][u] = v[u];
}

template <int R>
__device__ __forceinline__ void fl_get(const FlCache<R>& c, const float* p, const int64_t (&e)[R],
                                       const bool (&ok)[R], float4 dflt, float4 (&out)[R]) {
  bool hit = false;
#pragma unroll
  for (int sl = 0; sl < 4; ++sl) {
    if (!hit && c.p[sl] == p) {
      hit = true;
#pragma unroll
      for (int u = 0; u < R; ++u) out[u] = c.v[sl][u];
    }
  }
  if (!hit) {
#pragma unroll
    for (int u = 0; u < R; ++u) out[u] = ok[u] ? ld4(p, e[u]) : dflt;
  }
}

__device__ __forceinline__ void fl_prefetch(const float* p, int64_t e) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + e));
}

template <int R>
__device__ __forceinline__ void fl_prefetch_op(const EwOp& op, const int64_t (&e)[R], const bool (&ok)[R]) {
  for (int i = 0; i < op.nterm; ++i)
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) fl_prefetch(op.term[i], e[u]);
  for (int i = 0; i < op.nfac; ++i)
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) fl_prefetch(op.fac[i], e[u]);
  if (op.y)
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) fl_prefetch(op.y, e[u]);
  if (op.base)
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) fl_prefetch(op.base, e[u]);
}

template <int R>
__device__ __forceinline__ void fl_op(const EwOp& op, int width, const int64_t (&r)[R], const int64_t (&e)[R],
                                      int j, const bool (&ok)[R], const RingWrite& ring, bool has_acc,
                                      const float4 (&acc)[R], FlCache<R>& cache) {
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f), one = make_float4(1.f, 1.f, 1.f, 1.f);
  float4 v[R], t[R];
  const int kind = op.kind;
  if (kind == EW_CONST1) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      v[u] = one;
      if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, one);
    }
    fl_push(cache, op.out, v);
    return;
  }
  if (kind == EW_FWD_MUL) {
    fl_get(cache, op.fac[0], e, ok, zero, v);
    for (int i = 1; i < op.nfac; ++i) {
      fl_get(cache, op.fac[i], e, ok, zero, t);
#pragma unroll
      for (int u = 0; u < R; ++u) v[u] = mul4(v[u], t[u]);
    }
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, v[u]);
    fl_push(cache, op.out, v);
    return;
  }
  if (has_acc) {
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = acc[u];
  } else if (op.base) {
    fl_get(cache, op.base, e, ok, zero, v);
  } else {
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = zero;
  }
  for (int i = 0; i < op.nterm; ++i) {  // ascending sum, as ew_apply
    fl_get(cache, op.term[i], e, ok, zero, t);
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = add4(v[u], t[u]);
  }
  if (kind == EW_FWD_ADD) {
    for (int i = 0; i < op.nrank1; ++i) {
      const float4 w = ld4(op.r1w[i], j);
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const float sv = ok[u] ? op.r1src[i][r[u]] : 0.0f;
        v[u] = add4(v[u], make_float4(w.x * sv, w.y * sv, w.z * sv, w.w * sv));
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      v[u] = make_float4(act_apply(op.act, v[u].x), act_apply(op.act, v[u].y), act_apply(op.act, v[u].z),
                         act_apply(op.act, v[u].w));
      if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, v[u]);
    }
    fl_push(cache, op.out, v);
    return;
  }
  // EW_BWD
  if (op.act == ACT_SIGMOID || op.act == ACT_TANH) {
    fl_get(cache, op.y, e, ok, zero, t);
#pragma unroll
    for (int u = 0; u < R; ++u)
      v[u] = mul4(v[u], make_float4(act_deriv(op.act, t[u].x), act_deriv(op.act, t[u].y),
                                    act_deriv(op.act, t[u].z), act_deriv(op.act, t[u].w)));
  }
  if (op.inj) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      t[u] = (ok[u] && r[u] >= op.inj_row0) ? ld4(op.inj, (r[u] - op.inj_row0) * width + j) : zero;
      v[u] = add4(v[u], t[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < R; ++u)
    if (ok[u]) st4(op.out, e[u], v[u]);
  fl_push(cache, op.out, v);
  if (op.nfac == 0) return;
  float4 f[kMaxFac][R];
#pragma unroll
  for (int i = 0; i < kMaxFac; ++i) {
    if (i < op.nfac) {
      fl_get(cache, op.fac[i], e, ok, one, f[i]);
    } else {
#pragma unroll
      for (int u = 0; u < R; ++u) f[i][u] = one;
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxFac; ++i) {
    if (i >= op.nfac || !op.eps[i]) continue;
    float4 pv[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      pv[u] = v[u];
#pragma unroll
      for (int k = 0; k < kMaxFac; ++k)
        if (k != i) pv[u] = mul4(pv[u], f[k][u]);
      if (ok[u]) st4(op.eps[i], e[u], pv[u]);
    }
    fl_push(cache, op.eps[i], pv);
  }
}

// The job chains (op 0 of job j takes tile_s columns [j*bu, (j+1)*bu)) and the
// fused elementwise chains over rows [r_lo, r_hi) x units [u0, u0 + bu), one
// element group (R rows x 4 units) per thread at a time.
template <int R>
__device__ __forceinline__ void frame_chains_fused(const EwChain* chains, int J, int nch, const RingWrite* rings,
                                                   const float* tile_s, int ld, int m0, int u0, int bu, int N,
                                                   int r_lo, int r_hi, int tid) {
  const int ncols = min(bu, N - u0);
  if (ncols <= 0 || r_hi <= r_lo || ncols % 4) return;
  const int g4 = ncols / 4, lanes = 256 / g4 * g4;
  if (tid >= lanes) return;
  const int g = tid % g4, layer = tid / g4, layers = lanes / g4;
  const int j = u0 + 4 * g;
#pragma unroll 1
  for (int rb = r_lo + layer; rb < r_hi; rb += layers * R) {
    int64_t rr[R], e[R];
    bool ok[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int rl = rb + u * layers;
      ok[u] = rl < r_hi;
      rr[u] = m0 + (ok[u] ? rl : r_lo);
      e[u] = rr[u] * N + j;
    }
    for (int c = 0; c < nch; ++c)
      for (int k = 0; k < chains[c].nops; ++k) fl_prefetch_op<R>(chains[c].op[k], e, ok);
    FlCache<R> cache;
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) cache.p[sl] = nullptr;
    for (int c = 0; c < nch; ++c) {
      float4 a[R];
      const bool has_acc = c < J;
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int rl = rb + u * layers;
        a[u] = has_acc ? *reinterpret_cast<const float4*>(tile_s + (ok[u] ? rl : r_lo) * ld + c * bu + 4 * g)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int k = 0; k < chains[c].nops; ++k)
        fl_op<R>(chains[c].op[k], N, rr, e, j, ok, rings[c], has_acc && k == 0, a, cache);
    }
  }
}

// every chain of the set can take the fused 16-byte path
__device__ __forceinline__ bool chains_vec_ok(const EwChain* chains, int nch, int N) {
  for (int c = 0; c < nch; ++c)
    if (!chain_vec_ok(chains[c], N)) return false;
  return true;
}

// ---- LSTM cell chains: critical outputs first ------------------------------
// The host recognises the two chain sets of a peephole-LSTM SCC loop
// (FrameLoop::pattern; the builders' cell wiring, engine.py:405-413 / 568-576):
//   1 forward (tiles span both gate jobs, the cell update fused):
//     g_j = act(acc_j + pf_j), p_j = x_j * g_j (j = input / forget gate),
//     cell = act(p_a + p_b)
//   2 backward: d = acc + e(t+1) + pb;  (d1, e10, e11) = (d, d*f11, d*f10);
//     (d2, e20, e21) likewise; dg3 = e[k3] * f'(y3); dg4 = e[k4] * f'(y4).
// Every value of an element group stays in registers (no store -> load round
// trip); pass 0 stores only what the next frame's GEMM reads (cell(t), or the
// two gate deltas) before the frame barrier, pass 1 -- run by four dedicated
// store warps while the next frame's main loop runs -- recomputes the group
// and stores the rest.  Arithmetic and order are exactly ew_apply's.
__device__ __forceinline__ float4 act4(int act, float4 v) {
  return make_float4(act_apply(act, v.x), act_apply(act, v.y), act_apply(act, v.z), act_apply(act, v.w));
}
__device__ __forceinline__ float4 dact4(int act, float4 y) {
  return make_float4(act_deriv(act, y.x), act_deriv(act, y.y), act_deriv(act, y.z), act_deriv(act, y.w));
}

template <int R>
__device__ __forceinline__ void lstm_chains(int pattern, int pass, const EwChain* chains, const RingWrite* rings,
                                            const float* tile_s, int ld, int m0, int u0, int bu, int N, int r_lo,
                                            int r_hi, int tid, int nthr, const EwOp* tail = nullptr,
                                            const RingWrite* tail_ring = nullptr) {
  const int ncols = min(bu, N - u0);
  if (ncols <= 0 || r_hi <= r_lo) return;
  const int g4 = ncols / 4, lanes = nthr / g4 * g4;
  if (tid >= lanes) return;
  const int g = tid % g4, layer = tid / g4, layers = lanes / g4;
  const int j = u0 + 4 * g;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int rb = r_lo + layer; rb < r_hi; rb += layers * R) {
    int64_t rr[R], e[R];
    bool ok[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int rl = rb + u * layers;
      ok[u] = rl < r_hi;
      rr[u] = m0 + (ok[u] ? rl : r_lo);
      e[u] = rr[u] * N + j;
    }
    auto acc_of = [&](int c, float4 (&a)[R]) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int rl = rb + u * layers;
        a[u] = *reinterpret_cast<const float4*>(tile_s + (ok[u] ? rl : r_lo) * ld + c * bu + 4 * g);
      }
    };
    auto load = [&](const float* p, float4 (&v)[R]) {
#pragma unroll
      for (int u = 0; u < R; ++u) v[u] = ok[u] ? ld4(p, e[u]) : zero;
    };
    auto store = [&](const EwOp& op, const RingWrite& ring, const float4 (&v)[R]) {
#pragma unroll
      for (int u = 0; u < R; ++u)
        if (ok[u]) ring_store4(op.out, e[u], rr[u], N, op.out_is_ring, ring, v[u]);
    };
    auto store_to = [&](float* p, const float4 (&v)[R]) {
#pragma unroll
      for (int u = 0; u < R; ++u)
        if (ok[u]) st4(p, e[u], v[u]);
    };
    if (pattern == 1) {
      const EwOp& ew = chains[2].op[0];
      float4 pa[R], pb[R];
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        const EwOp& o0 = chains[jb].op[0];
        const EwOp& o1 = chains[jb].op[1];
        float4 a[R], t[R], x[R], gt[R], pr[R];
        acc_of(jb, a);
        load(o0.term[0], t);
        const int gi = o1.fac[0] == o0.out ? 0 : 1;
        load(o1.fac[1 - gi], x);
#pragma unroll
        for (int u = 0; u < R; ++u) {
          gt[u] = act4(o0.act, add4(a[u], t[u]));
          pr[u] = gi == 0 ? mul4(gt[u], x[u]) : mul4(x[u], gt[u]);
        }
        if (pass == 1) {
          store(o0, rings[jb], gt);
          store(o1, rings[jb], pr);
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
          if (jb == 0) pa[u] = pr[u];
          else pb[u] = pr[u];
        }
      }
      if (pass == 1 && tail) {  // the fused step after the loop: act(0 + cell(t))
        const bool a_first = ew.term[0] == chains[0].op[1].out;
        float4 v[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const float4 t0 = a_first ? pa[u] : pb[u], t1 = a_first ? pb[u] : pa[u];
          v[u] = act4(tail->act, add4(zero, act4(ew.act, add4(add4(zero, t0), t1))));
        }
#pragma unroll
        for (int u = 0; u < R; ++u)
          if (ok[u]) ring_store4(tail->out, e[u], rr[u], N, tail->out_is_ring, *tail_ring, v[u]);
      }
      if (pass == 0) {
        const bool a_first = ew.term[0] == chains[0].op[1].out;
        float4 c[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const float4 t0 = a_first ? pa[u] : pb[u], t1 = a_first ? pb[u] : pa[u];
          c[u] = act4(ew.act, add4(add4(zero, t0), t1));
        }
        store(ew, rings[2], c);
      }
    } else {
      const EwOp* o = chains[0].op;
      float4 a[R], t0[R], t1[R];
      acc_of(0, a);
      load(o[0].term[0], t0);
      load(o[0].term[1], t1);
      float4 d0[R];
#pragma unroll
      for (int u = 0; u < R; ++u) d0[u] = add4(add4(a[u], t0[u]), t1[u]);
      float4 f10[R], f11[R], f20[R], f21[R];
      load(o[1].fac[0], f10);
      load(o[1].fac[1], f11);
      load(o[2].fac[0], f20);
      load(o[2].fac[1], f21);
      float4 d1[R], e10[R], e11[R], d2[R], e20[R], e21[R];
#pragma unroll
      for (int u = 0; u < R; ++u) {
        d1[u] = add4(zero, d0[u]);
        e10[u] = mul4(d1[u], f11[u]);
        e11[u] = mul4(d1[u], f10[u]);
        d2[u] = add4(zero, d0[u]);
        e20[u] = mul4(d2[u], f21[u]);
        e21[u] = mul4(d2[u], f20[u]);
      }
      if (pass == 0) {
        // the two gate deltas: eps k of ops 1 / 2 through f' of their y
#pragma unroll
        for (int q = 3; q <= 4; ++q) {
          const float* src = o[q].term[0];
          float4 y[R], v[R];
          load(o[q].y, y);
#pragma unroll
          for (int u = 0; u < R; ++u) {
            const float4 s = src == o[1].eps[0] ? e10[u] : src == o[1].eps[1] ? e11[u]
                           : src == o[2].eps[0] ? e20[u] : e21[u];
            v[u] = mul4(add4(zero, s), dact4(o[q].act, y[u]));
          }
          store_to(o[q].out, v);
        }
      } else {
        store_to(o[0].out, d0);
        store_to(o[1].out, d1);
        store_to(o[1].eps[0], e10);
        store_to(o[1].eps[1], e11);
        store_to(o[2].out, d2);
        store_to(o[2].eps[0], e20);
        store_to(o[2].eps[1], e21);
        if (tail) {  // the fused step after the loop: (0 + eps) * f'(y)
          const float* src = tail->term[0];
          float4 y[R], v[R];
          load(tail->y, y);
#pragma unroll
          for (int u = 0; u < R; ++u) {
            const float4 s = src == o[1].eps[0] ? e10[u] : src == o[1].eps[1] ? e11[u]
                           : src == o[2].eps[0] ? e20[u] : e21[u];
            v[u] = mul4(add4(zero, s), dact4(tail->act, y[u]));
          }
          store_to(tail->out, v);
        }
      }
    }
  }
}

// Pass 0 of lstm_chains split in two around the split-K reduction: every
// operand that does not come from the accumulator (hoisted pre-activations,
// gate outputs, cell(t-1) stored one frame earlier, the eps the store warps
// wrote behind the previous barrier) is copied into shared memory by bulk
// copies (one per operand row) first, so the loads overlap the DSMEM
// reduction; the second half reads the reduced accumulator, evaluates two row
// groups at a time and stores.  Operand k's slab (rows [r_lo, r_hi) x the
// tile's units) is the pipeline's A region (even k) or B_lo region (odd k) of
// stage k / 2: idle from the frame's last MMA until the next frame's A loads
// (which wait for this CTA's barrier arrival) and conversions (done by these
// same threads).  Same operands and arithmetic order as lstm_chains pass 0.
#ifndef RGB_FL_POST_U
#define RGB_FL_POST_U 2
#endif
__device__ __forceinline__ int lstm_nops(int pattern) { return pattern == 1 ? 4 : 6; }

template <int SLAB>
__device__ __forceinline__ bool lstm_pre_ok(int bu, int N, int u0, int r_lo, int r_hi) {
  const int ncols = min(bu, N - u0);
  if (ncols <= 0 || r_hi <= r_lo) return true;  // nothing to do
  return ncols % 4 == 0 && N % 4 == 0 && u0 % 4 == 0 && (r_hi - r_lo) * ncols * 4 <= SLAB;
}

__device__ __forceinline__ const float* lstm_bwd_fac(const EwOp* o, int q) {
  const float* src = o[q].term[0];
  return src == o[1].eps[0] ? o[1].fac[1] : src == o[1].eps[1] ? o[1].fac[0]
       : src == o[2].eps[0] ? o[2].fac[1] : o[2].fac[0];
}

__device__ __forceinline__ const float* lstm_operand(int pattern, const GemmGroup& pg, int k) {
  if (pattern == 1) {
    const EwOp &o0 = pg.job[k >> 1].epi.op[0], &o1 = pg.job[k >> 1].epi.op[1];
    return (k & 1) ? o1.fac[o1.fac[0] == o0.out ? 1 : 0] : o0.term[0];
  }
  const EwOp* o = pg.job[0].epi.op;
  switch (k) {
    case 0: return o[0].term[0];
    case 1: return o[0].term[1];
    case 2: return lstm_bwd_fac(o, 3);
    case 3: return lstm_bwd_fac(o, 4);
    case 4: return o[3].y;
    default: return o[4].y;
  }
}

template <int STAGE_BYTES, int A_BYTES, int B_BYTES>
__device__ __forceinline__ uint32_t lstm_slab(uint32_t pipe, int k) {
  return pipe + (k >> 1) * STAGE_BYTES + ((k & 1) ? A_BYTES + B_BYTES : 0);
}

// the store warps: 16-byte cp.async of every operand element group, arriving
// on `full` (count nthr) when this thread's copies have landed
template <int STAGE_BYTES, int A_BYTES, int B_BYTES>
__device__ __forceinline__ void lstm_pre(int pattern, const GemmGroup& pg, int m0, int u0, int bu, int N, int r_lo,
                                         int r_hi, int tid, int nthr, uint32_t pipe, uint64_t* full) {
  const int ncols = max(0, min(bu, N - u0)), rows = max(0, r_hi - r_lo), np = lstm_nops(pattern);
  const int g4 = ncols / 4, per_k = rows * g4;
  const uint32_t row_bytes = (uint32_t)ncols * 4u;
  const float* ptr[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) ptr[k] = k < np ? lstm_operand(pattern, pg, k) : nullptr;
  for (int it = tid; it < np * per_k; it += nthr) {
    const int k = it / per_k, rem = it - k * per_k, r = rem / g4, c4 = rem - r * g4;
    const float* src = ptr[k] + ((int64_t)(m0 + r_lo + r) * N + u0 + 4 * c4);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(lstm_slab<STAGE_BYTES, A_BYTES, B_BYTES>(pipe, k) +
                                                                    (uint32_t)r * row_bytes + 16u * c4),
                 "l"(__cvta_generic_to_global(src))
                 : "memory");
  }
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(full)) : "memory");
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

template <int STAGE_BYTES, int A_BYTES, int B_BYTES>
__device__ __forceinline__ void lstm_post(int pattern, const EwChain* chains, const RingWrite* rings,
                                          const float* tile_s, int ld, int m0, int u0, int bu, int N, int r_lo,
                                          int r_hi, int tid, int nthr, uint32_t pipe) {
  const int ncols = min(bu, N - u0);
  if (ncols <= 0 || r_hi <= r_lo) return;
  const int g4 = ncols / 4, lanes = nthr / g4 * g4;
  if (tid >= lanes) return;
  const int g = tid % g4, layer = tid / g4, layers = lanes / g4;
  const int j = u0 + 4 * g;
  const uint32_t row_bytes = (uint32_t)ncols * 4u;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const EwOp* o = chains[0].op;
  auto v = [&](int rl, int k) {
    return lds4(lstm_slab<STAGE_BYTES, A_BYTES, B_BYTES>(pipe, k) + (uint32_t)(rl - r_lo) * row_bytes + 16u * g);
  };
  constexpr int U = RGB_FL_POST_U;  // row groups in flight per thread
#pragma unroll 1
  for (int rb = r_lo + layer; rb < r_hi; rb += U * layers) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int rq = rb + u * layers;
      const bool ok = rq < r_hi;
      const int rl = ok ? rq : rb;
      const int64_t rr = m0 + rl, e = rr * N + j;
      if (pattern == 1) {
        const EwOp& ew = chains[2].op[0];
        float4 pr[2];
#pragma unroll
        for (int jb = 0; jb < 2; ++jb) {
          const EwOp &o0 = chains[jb].op[0], &o1 = chains[jb].op[1];
          const float4 a = *reinterpret_cast<const float4*>(tile_s + rl * ld + jb * bu + 4 * g);
          const float4 gt = act4(o0.act, add4(a, v(rl, 2 * jb)));
          pr[jb] = o1.fac[0] == o0.out ? mul4(gt, v(rl, 2 * jb + 1)) : mul4(v(rl, 2 * jb + 1), gt);
        }
        const bool a_first = ew.term[0] == chains[0].op[1].out;
        const float4 t0 = a_first ? pr[0] : pr[1], t1 = a_first ? pr[1] : pr[0];
        const float4 c = act4(ew.act, add4(add4(zero, t0), t1));
        if (ok) ring_store4(ew.out, e, rr, N, ew.out_is_ring, rings[2], c);
      } else {
        const float4 a = *reinterpret_cast<const float4*>(tile_s + rl * ld + 4 * g);
        const float4 d = add4(zero, add4(add4(a, v(rl, 0)), v(rl, 1)));
#pragma unroll
        for (int q = 3; q <= 4; ++q) {
          const float4 s = mul4(d, v(rl, q - 1));
          const float4 w = mul4(add4(zero, s), dact4(o[q].act, v(rl, q + 1)));
          if (ok) st4(o[q].out, e, w);
        }
      }
    }
  }
}

// Sums rows [r_lo, r_hi) of the csplit partial tiles of a cluster (DSMEM,
// split order) into this CTA's tile_s; NB remote loads per thread in flight
// (a DSMEM round trip is ~200 cycles; serial loads made this 3.5 us).
template <int G4, int NB>
__device__ __forceinline__ void reduce_split_rows(float* tile_s, int ld, int r_lo, int r_hi, int csplit, int tid) {
  const int nq = (r_hi - r_lo) * G4;
  for (int q0 = tid; q0 < nq; q0 += 256 * NB) {
    float4 a[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int q = q0 + 256 * i;
      const int off = (r_lo + q / G4) * ld + (q % G4) * 4;
      a[i] = q < nq ? ld_dsmem4(tile_s + off, 0u) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int k = 1; k < csplit; ++k) {
      float4 b[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int q = q0 + 256 * i;
        const int off = (r_lo + q / G4) * ld + (q % G4) * 4;
        b[i] = q < nq ? ld_dsmem4(tile_s + off, (uint32_t)k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) a[i] = add4(a[i], b[i]);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int q = q0 + 256 * i;
      if (q < nq) *reinterpret_cast<float4*>(tile_s + (r_lo + q / G4) * ld + (q % G4) * 4) = a[i];
    }
  }
}

// A chain over rows [r_lo, r_hi) x units [u0, u0 + bu) of the tile; with
// `acc`, op 0 takes the staged accumulator columns [c0, c0 + bu) of tile_s.
// 16-byte groups, R rows per thread and pass (one operand latency per op
// covers R rows); scalar fallback for unaligned chains.
template <int R>
__device__ __forceinline__ void frame_chain(const EwChain& ch, const float* tile_s, int ld, int c0, bool acc,
                                            int m0, int u0, int bu, int N, int r_lo, int r_hi,
                                            const RingWrite& ring, int tid) {
  const int ncols = min(bu, N - u0);
  if (ncols <= 0 || r_hi <= r_lo) return;
  if (chain_vec_ok(ch, N) && ncols % 4 == 0) {
    const int g4 = ncols / 4, lanes_per_layer = 256 / g4 * g4;
    if (tid >= lanes_per_layer) return;
    const int g = tid % g4, layer = tid / g4, layers = lanes_per_layer / g4;
#pragma unroll 1
    for (int rb = r_lo + layer; rb < r_hi; rb += layers * R) {
      int64_t rr[R];
      bool ok[R];
      float4 a[R];
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int rl = rb + u * layers;
        ok[u] = rl < r_hi;
        rr[u] = m0 + (ok[u] ? rl : r_lo);
        a[u] = acc ? *reinterpret_cast<const float4*>(tile_s + (ok[u] ? rl : r_lo) * ld + c0 + 4 * g)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#ifdef RGB_FL_TRACE
      for (int k = 0; k < ch.nops; ++k) {
        ew_apply_vec_variant<R>(ch.op[k], N, rr, u0 + 4 * g, ok, ring, acc && k == 0, a);
        if (tid == 0 && k < 6) fl_mark(g_fl_frame, 8 + k);
      }
#ifdef RGB_FL_TRACE2
      // the same ops again (idempotent): warm-cache / warm-TLB latency per op
      for (int k = 0; k < ch.nops; ++k) {
        ew_apply_vec_variant<R>(ch.op[k], N, rr, u0 + 4 * g, ok, ring, acc && k == 0, a);
        if (tid == 0 && k < 2) fl_mark(g_fl_frame, 14 + k);
      }
#endif
#else
      ew_chain_vec<R>(ch, N, rr, u0 + 4 * g, ok, ring, acc, a);
#endif
    }
    return;
  }
  for (int e = tid; e < (r_hi - r_lo) * ncols; e += 256) {
    const int rl = r_lo + e / ncols, cl = e % ncols;
    const float a = acc ? tile_s[rl * ld + c0 + cl] : 0.0f;
    for (int k = 0; k < ch.nops; ++k) ew_apply(ch.op[k], N, m0 + rl, u0 + cl, ring, acc && k == 0, a);
  }
}


// Tiles: 128 stream rows x `bu` units of EVERY job of the GEMM step (the jobs
// share the A operand, e.g. cell(t-1) feeding the input and forget gates), so
// one MMA of N = njobs * bu covers them all and the step's elementwise ops
// (the cell update reading both gates' products) are element-local to the
// tile: they run in the epilogue instead of behind another grid barrier.
constexpr int kFrameThreads = 512;  // warps 0-7 convert + epilogue, 8 / 10 TMA, 9 MMA, 11 L2 prefetch, 12-15 stores

template <int BN>
__global__ void __launch_bounds__(kFrameThreads, 1)
    tma_frame_loop_kernel(const __grid_constant__ FrameLoop fl, const __grid_constant__ GemmGroup p) {
  using C = FCfg<BN>;
  constexpr int BK = C::BK;
  constexpr int NST = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* tile_s = reinterpret_cast<float*>(smem + NST * C::STAGE_BYTES);
  uint64_t* tma_full = reinterpret_cast<uint64_t*>(smem + NST * C::STAGE_BYTES + C::TILE_BYTES);
  uint64_t* conv_full = tma_full + 8;
  uint64_t* empty = conv_full + 8;
  uint64_t* done = empty + 8;            // MMA of a frame complete
  uint64_t* acc_empty = done + 1;        // epilogue has read the accumulator
  uint64_t* part_ready = acc_empty + 1;  // split-K: partial tiles of the cluster staged
  uint64_t* read_done = part_ready + 1;  // split-K: peers finished reading this CTA's tile
  uint64_t* st_go = read_done + 1;       // LSTM patterns: pass 1 of a frame may start
  uint64_t* st_done = st_go + 1;         // LSTM patterns: pass 1 of a frame is done
  uint64_t* pre_full = st_done + 1;      // LSTM patterns: the frame's chain operands are in shared memory
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pre_full + 1);
  EwChain* chains = reinterpret_cast<EwChain*>(smem + NST * C::STAGE_BYTES + C::TILE_BYTES + 512);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int splits = p.splits > 1 ? p.splits : 1;
  const int split = blockIdx.x % splits, tile_lin = blockIdx.x / splits;
  const int csplit = p.csplit ? splits : 1;
  const int J = p.njobs, bu = fl.bu;
  const int ublocks = (p.job[0].n + bu - 1) / bu;
  const int m0 = (tile_lin / ublocks) * BM, u0 = (tile_lin % ublocks) * bu;
  const int M = p.rows, N = p.job[0].n;
  const int box = bu == 32 ? 0 : (bu == 64 ? 1 : (bu == 128 ? 2 : 3));
  int nstages = 0;
  for (int sg = 0; sg < p.job[0].nseg; ++sg) nstages += (p.job[0].seg[sg].k + BK - 1) / BK;
  const int s_begin = (int)((long long)split * nstages / splits);
  nstages = (int)((long long)(split + 1) * nstages / splits) - s_begin;
  const unsigned nbar = 1u + (fl.fuse_ew ? 0u : (unsigned)fl.n_ew);  // grid barriers per frame

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&tma_full[s], 2);
      mbar_init(&conv_full[s], kProducers);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(acc_empty, 1);
    mbar_init(part_ready, csplit);
    mbar_init(read_done, csplit);
    mbar_init(st_go, 1);
    mbar_init(st_done, 1);
    mbar_init(pre_full, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // the barrier generation at launch; every CTA reads it before its first
  // arrival, and no barrier completes before every CTA arrived
  const unsigned gen0 = *reinterpret_cast<volatile unsigned*>(fl.bar + 1);  // counter base of this launch
  const unsigned nblk = gridDim.x;
  auto bar_target = [&](unsigned k) { return gen0 + k * nblk; };  // barrier k (1-based) complete
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (csplit > 1) cluster_sync();
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  // registers: the converter / epilogue warp groups get 168, the producer
  // group 48, the store group keeps 128 (2 x 128 x 168 + 128 x 48 + 128 x 128 = 64K)
  if (warp >= 12) {
    // ---- LSTM patterns: pass 1 (the non-critical outputs) of each frame,
    // overlapping the next frame's main loop ----
    if (fl.pattern) {
    const int stid = threadIdx.x - 384;
    const int rlo = csplit > 1 ? split * BM / csplit : 0;
    const int rhi = min(csplit > 1 ? (split + 1) * BM / csplit : BM, M - m0);
    const bool use_pre = NST >= 3 && fl.preload && lstm_pre_ok<(C::A_BYTES < C::B_BYTES ? C::A_BYTES : C::B_BYTES)>(bu, N, u0, rlo, rhi);
    const uint32_t pipe = smem_u32(smem);
    for (int f = 0; f <= fl.nframes; ++f) {
      if (f > 0) {  // pass 1 of frame f - 1
        mbar_wait(st_go, (f - 1) & 1);
        const GemmGroup& pf = fl.frames[f - 1];
        RingWrite rings[3] = {pf.ring, pf.ring, fl.n_ew ? fl.ew[(size_t)(f - 1) * fl.n_ew].ring : pf.ring};
        const EwOp* tail = fl.tail ? &fl.tail[f - 1].chain[0].op[0] : nullptr;
        const RingWrite tring = fl.tail ? fl.tail[f - 1].ring : pf.ring;
        lstm_chains<2>(fl.pattern, 1, chains, rings, tile_s, C::EPI_LD, m0, u0, bu, N, rlo, rhi, stid, 128, tail,
                       &tring);
        asm volatile("bar.sync 5, 128;" ::: "memory");
        if (stid == 0) mbar_arrive(st_done);
      }
      if (use_pre && f < fl.nframes) {  // frame f's chain operands, once its MMAs are done with the slabs
        mbar_wait(done, f & 1);
        lstm_pre<C::STAGE_BYTES, C::A_BYTES, C::B_BYTES>(fl.pattern, fl.frames[f], m0, u0, bu, N, rlo, rhi, stid,
                                                          128, pipe, pre_full);
      }
    }
    }
  } else if (warp < 12) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 48;");
  if (warp == 11) {
    if (fl.prefetch) {
    // ---- L2 prefetch of frame f's epilogue operands (the chains' inputs that
    // do not come from the accumulator: hoisted partials, gate activations,
    // delayed state, co-factors, ...) while the main loop runs: the chains
    // are latency-bound on these loads (~1-2 us per op from HBM)
    for (int f = 0; f < fl.nframes; ++f) {
      if (f > 0) ctr_wait(fl.bar, bar_target((unsigned)f * nbar));
      const GemmGroup& pf = fl.frames[f];
      const int rlo = csplit > 1 ? split * BM / csplit : 0, rhi = min(csplit > 1 ? (split + 1) * BM / csplit : BM, M - m0);
      const int bytes = min(bu, N - u0) * 4;
      if (bytes <= 0 || (bytes & 15)) continue;
      const int nch = J + (fl.fuse_ew ? fl.n_ew : 0);
      int slot = 0;
      for (int c = 0; c < nch; ++c) {
        const EwChain& ch = c < J ? pf.job[c].epi : fl.ew[(size_t)f * fl.n_ew + (c - J)].chain[0];
        for (int k = 0; k < ch.nops; ++k) {
          const EwOp& o = ch.op[k];
          const float* ptrs[kMaxTerms + kMaxFac + 2];
          int np = 0;
          for (int i = 0; i < o.nterm; ++i) ptrs[np++] = o.term[i];
          for (int i = 0; i < o.nfac; ++i) ptrs[np++] = o.fac[i];
          if (o.y) ptrs[np++] = o.y;
          if (o.base) ptrs[np++] = o.base;
          for (int i = 0; i < np; ++i) {
            for (int rr = rlo; rr < rhi; ++rr, ++slot) {
              if ((slot & 31) != lane) continue;
              const float* a = ptrs[i] + ((int64_t)(m0 + rr) * N + u0);
              if (reinterpret_cast<uintptr_t>(a) & 15) continue;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
            }
          }
        }
      }
    }
    }
  } else if (warp == 8 || warp == 10) {
    if (lane == 0) {
      // ---- TMA: warp 8 loads the state operand A (after the frame barrier),
      // warp 10 the weights B of every job (frame independent: runs ahead)
      const bool load_a = warp == 8;
      int g = 0;
      for (int f = 0; f < fl.nframes; ++f) {
        const GemmGroup& pf = fl.frames[f];
        if (load_a && f > 0) {
          ctr_wait(fl.bar, bar_target((unsigned)f * nbar));
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        if (load_a) FL_MARK(f, 0);
        int seg = 0, k0 = 0;
        for (int skip = s_begin; skip > 0;) {
          const int ns = (pf.job[0].seg[seg].k + BK - 1) / BK;
          if (skip >= ns) {
            skip -= ns;
            ++seg;
          } else {
            k0 = skip * BK;
            skip = 0;
          }
        }
        for (int it = 0; it < nstages; ++it, ++g) {
          const int s = g % NST;
          mbar_wait(&empty[s], ((g / NST) & 1) ^ 1);
          uint8_t* base = smem + s * C::STAGE_BYTES;
          mbar_expect_tx(&tma_full[s], load_a ? C::A_BYTES : C::B_BYTES);
          if (load_a) {
            tma_load_2d(base, pf.job[0].seg[seg].ta, k0, pf.job[0].seg[seg].arow + m0, &tma_full[s]);
          } else {
            for (int j = 0; j < J; ++j)  // job j's bu weight rows land at rows [j*bu, (j+1)*bu) of B
              tma_load_2d(base + C::A_BYTES + j * bu * 128, map_at(pf.job[j].seg[seg].tb, box), k0, u0,
                          &tma_full[s]);
          }
          k0 += BK;
          if (k0 >= pf.job[0].seg[seg].k) {
            k0 = 0;
            ++seg;
          }
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      // ---- MMA issuer: A hi / lo from TMEM, B from shared memory ----
      const uint32_t idesc = idesc_tf32(BM, BN, 0, 0);
      const bool split3 = p.terms != 1;
      int g = 0;
      for (int f = 0; f < fl.nframes; ++f) {
        if (f > 0) mbar_wait(acc_empty, (f - 1) & 1);
        for (int it = 0; it < nstages; ++it, ++g) {
          const int s = g % NST;
          mbar_wait(&conv_full[s], (g / NST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t b_hi = smem_u32(smem + s * C::STAGE_BYTES) + C::A_BYTES, b_lo = b_hi + C::B_BYTES;
          const uint32_t ta_hi = tmem + BN + 64 * s, ta_lo = ta_hi + 32;
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {
            const uint64_t dbh = smem_desc(b_hi + j * 32, 16, 1024, 2), dbl = smem_desc(b_lo + j * 32, 16, 1024, 2);
            const uint32_t acc0 = (it > 0 || j > 0) ? 1u : 0u;
            if (split3) {
              mma_tf32_ta(tmem, ta_lo + 8 * j, dbh, idesc, acc0);
              mma_tf32_ta(tmem, ta_hi + 8 * j, dbl, idesc, 1u);
            }
            mma_tf32_ta(tmem, ta_hi + 8 * j, dbh, idesc, split3 ? 1u : acc0);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(done);
      }
    }
  }
  }
  if (warp < 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 168;");
    // ---- warps 0-7: converters, then per frame the epilogue and the
    // elementwise steps ----
    const int tid = threadIdx.x;
    const int quarter = warp & 3, kh = warp >> 2, r = quarter * 32 + lane;
    int g = 0;
    for (int f = 0; f < fl.nframes; ++f) {
      const GemmGroup& pf = fl.frames[f];
      for (int it = 0; it < nstages; ++it, ++g) {
        const int s = g % NST;
        mbar_wait(&tma_full[s], (g / NST) & 1);
        uint8_t* base = smem + s * C::STAGE_BYTES;
        {
          const uint8_t* arow = base + r * 128;
          float hi[16], lo[16];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c = kh * 4 + cc;
            const float4 x = *reinterpret_cast<const float4*>(arow + ((c ^ (r & 7)) * 16));
            hi[4 * cc] = x.x, hi[4 * cc + 1] = x.y, hi[4 * cc + 2] = x.z, hi[4 * cc + 3] = x.w;
          }
          if (p.terms != 1) {
#pragma unroll
            for (int q = 0; q < 16; ++q) lo[q] = tf32_residual(hi[q]);
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) hi[q] = tf32_rna(hi[q]);
          }
          const uint32_t ta = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + BN + 64 * s + 16 * kh;
          tmem_st16(ta, hi);
          if (p.terms != 1) tmem_st16(ta + 32, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        }
        if (p.terms != 1) {
          const float4* b_hi = reinterpret_cast<const float4*>(base + C::A_BYTES);
          float4* b_lo = reinterpret_cast<float4*>(base + C::A_BYTES + C::B_BYTES);
          for (int q = tid; q < C::B_BYTES / 16; q += kProducers) {
            const float4 x = b_hi[q];
            b_lo[q] = make_float4(tf32_residual(x.x), tf32_residual(x.y), tf32_residual(x.z), tf32_residual(x.w));
          }
        } else {
          round_tf32_inplace(base + C::A_BYTES, C::B_BYTES, tid, kProducers);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&conv_full[s]);
      }
      // ---- epilogue of frame f ----
      if (fl.pattern && f > 0) mbar_wait(st_done, (f - 1) & 1);  // pass 1 of f-1 done with tile_s / chains
      for (int j = 0; j < J; ++j) stage_chain(&chains[j], pf.job[j].epi, tid, 256);
      if (fl.fuse_ew)
        for (int e = 0; e < fl.n_ew; ++e) stage_chain(&chains[J + e], fl.ew[(size_t)f * fl.n_ew + e].chain[0], tid, 256);
      // the rows this CTA finishes (split-K: its slice of the reduced tile)
      const int r_lo = csplit > 1 ? split * BM / csplit : 0, r_hi = csplit > 1 ? (split + 1) * BM / csplit : BM;
      const int rows_hi = min(r_hi, M - m0);
      const uint32_t pipe = smem_u32(smem);
      const bool use_pre = NST >= 3 && fl.pattern && fl.preload &&
                           lstm_pre_ok<(C::A_BYTES < C::B_BYTES ? C::A_BYTES : C::B_BYTES)>(bu, N, u0, r_lo, rows_hi);
      if (csplit > 1 && f > 0) mbar_wait_cluster(read_done, (f - 1) & 1);  // peers done with tile_s
      mbar_wait(done, f & 1);
      if (tid == 0) FL_MARK(f, 1);
      // acquire the frame barrier the A loads waited on: the chains read
      // operands other SMs stored in earlier frames (no stale L1 lines)
      if (f > 0) (void)ld_acquire_u32(fl.bar);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      {  // accumulator -> tile_s (warp w: TMEM lane quarter w%4, column half w/4)
        const int half = warp >> 2, r_loc = quarter * 32 + lane;
        for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 16) {
          float v[16];
          tmem_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cc, v);
          float4* dst = reinterpret_cast<float4*>(tile_s + r_loc * C::EPI_LD + cc);
          dst[0] = make_float4(v[0], v[1], v[2], v[3]);
          dst[1] = make_float4(v[4], v[5], v[6], v[7]);
          dst[2] = make_float4(v[8], v[9], v[10], v[11]);
          dst[3] = make_float4(v[12], v[13], v[14], v[15]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tid == 0) mbar_arrive(acc_empty);
      if (tid == 0) FL_MARK(f, 2);
      if (csplit > 1) {
        // this CTA sums rows [r_lo, r_hi) of the cluster's partial tiles in split order
        if (tid < csplit) mbar_arrive_cluster(part_ready, (uint32_t)tid);
        mbar_wait_cluster(part_ready, f & 1);
        reduce_split_rows<BN / 4, 8>(tile_s, C::EPI_LD, r_lo, r_hi, csplit, tid);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (tid < csplit) mbar_arrive_cluster(read_done, (uint32_t)tid);
      }
      if (tid == 0) FL_MARK(f, 3);
#ifdef RGB_FL_TRACE
      if (tid == 0 && blockIdx.x == 0) g_fl_frame = f;
#endif
      const int nch = J + (fl.fuse_ew ? fl.n_ew : 0);
      if (fl.pattern) {
        RingWrite rings[3] = {pf.ring, pf.ring, fl.n_ew ? fl.ew[(size_t)f * fl.n_ew].ring : pf.ring};
        if (use_pre) {
          mbar_wait(pre_full, f & 1);  // the store warps' copies of the chain operands
          if (tid == 0) FL_MARK(f, 7);
          lstm_post<C::STAGE_BYTES, C::A_BYTES, C::B_BYTES>(fl.pattern, chains, rings, tile_s, C::EPI_LD, m0, u0,
                                                             bu, N, r_lo, rows_hi, tid, 256, pipe);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the next frame's TMA reuses the slabs
        } else
          lstm_chains<2>(fl.pattern, 0, chains, rings, tile_s, C::EPI_LD, m0, u0, bu, N, r_lo, rows_hi, tid, 256);
      } else if (fl.forward && chains_vec_ok(chains, nch, N) && min(bu, N - u0) % 4 == 0) {
        RingWrite rings[4];
        for (int c = 0; c < nch; ++c) rings[c] = c < J ? pf.ring : fl.ew[(size_t)f * fl.n_ew + (c - J)].ring;
        frame_chains_fused<2>(chains, J, nch, rings, tile_s, C::EPI_LD, m0, u0, bu, N, r_lo, rows_hi, tid);
      } else {
#ifndef RGB_FL_R
#define RGB_FL_R 4
#endif
        for (int j = 0; j < J; ++j)
          frame_chain<RGB_FL_R>(chains[j], tile_s, C::EPI_LD, j * bu, true, m0, u0, bu, N, r_lo, rows_hi, pf.ring,
                                tid);
        if (fl.fuse_ew) {
          // the step's elementwise ops read the job chains' outputs at the same
          // (row, unit): visible to the CTA after the barrier
          for (int e = 0; e < fl.n_ew; ++e) {
            asm volatile("bar.sync 1, 256;" ::: "memory");
            frame_chain<4>(chains[J + e], tile_s, C::EPI_LD, 0, false, m0, u0, bu, N, r_lo, rows_hi,
                           fl.ew[(size_t)f * fl.n_ew + e].ring, tid);
          }
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tid == 0) FL_MARK(f, 4);
      if (tid == 0) ctr_arrive(fl.bar);
      if (fl.pattern && tid == 0) mbar_arrive(st_go);  // the store warps take the rest of the frame
      // ---- unfused elementwise steps of frame f (all CTAs, between grid barriers) ----
      for (int e = 0; e < (fl.fuse_ew ? 0 : fl.n_ew); ++e) {
        const EwLaunch& L = fl.ew[(size_t)f * fl.n_ew + e];
        if (tid == 0) ctr_wait(fl.bar, bar_target((unsigned)f * nbar + 1u + (unsigned)e));
        asm volatile("bar.sync 1, 256;" ::: "memory");
        (void)ld_acquire_u32(fl.bar);  // every thread: acquire before reading other SMs' stores
        if (tid == 0) FL_MARK(f, 5);
        for (int c = 0; c < L.nchains; ++c) {
          stage_chain(&chains[0], L.chain[c], tid, 256);
          asm volatile("bar.sync 1, 256;" ::: "memory");
          const EwChain& ch = chains[0];
          if (chain_vec_ok(ch, ch.width)) {
            const uint32_t w4 = (uint32_t)(ch.width / 4);
            const uint32_t nq = (uint32_t)L.rows * w4;
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
            for (uint32_t q = blockIdx.x * 256u + tid; q < nq; q += gridDim.x * 256u) {
              const uint32_t r32 = q / w4;
              const int64_t rr[1] = {(int64_t)r32};
              const bool ok[1] = {true};
              const float4 acc[1] = {zero};
              ew_chain_vec<1>(ch, ch.width, rr, (int)(q - r32 * w4) * 4, ok, L.ring, false, acc);
            }
          } else {
            const int64_t total = (int64_t)L.rows * ch.width;
            for (int64_t q = (int64_t)blockIdx.x * 256 + tid; q < total; q += (int64_t)gridDim.x * 256) {
              const int64_t rr = q / ch.width;
              const int j = (int)(q - rr * ch.width);
              for (int k = 0; k < ch.nops; ++k) ew_apply(ch.op[k], ch.width, rr, j, L.ring, false, 0.0f);
            }
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
        }
        if (tid == 0) FL_MARK(f, 6);
        if (tid == 0) ctr_arrive(fl.bar);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (csplit > 1) cluster_sync();  // peers' last DSMEM reads of this CTA's tile are done
  else __syncthreads();
  if (warp == 9) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  if (threadIdx.x == 0) ctr_finish(fl.bar, bar_target((unsigned)fl.nframes * nbar), nblk);
}

// Widest N tile that still gives most of the 148 SMs a tile.
template <class F>
int pick_bn(F tiles_for) {
  static int forced = -1;  // RGB_TC_BN: tile-width override for tuning experiments
  if (forced < 0) {
    const char* e = getenv("RGB_TC_BN");
    forced = e ? atoi(e) : 0;
  }
  if (forced == 32 || forced == 64 || forced == 128 || forced == 256) return forced;
  for (int bn : {256, 128, 64})
    if (tiles_for(bn) >= 120) return bn;
  return 32;
}

}  // namespace tc

namespace {

int g_tc_terms = 3;  // 3: 3xTF32 (fp32-exact, default); 1: plain TF32 (rgb_set_tc_precision)
int g_tc_opt[3] = {-1, -1, -1};  // pair, persistent, cluster split-K (-1: from the environment)

bool pair_enabled() {  // RGB_TC_PAIR=0 disables the CTA-pair kernels (tuning experiments); rgb_set_tc_config overrides
  int& on = g_tc_opt[0];
  if (on < 0) {
    const char* e = getenv("RGB_TC_PAIR");
    on = e ? atoi(e) != 0 : 1;
  }
  return on == 1;
}

// Full-machine pair tiles pay in 3xTF32 only (they halve the B residual
// conversion per CTA).  Plain TF32 has no conversion and the pair's cross-CTA
// handshake becomes the bound: single CTAs measured 1.5-1.7x faster on the
// hoisted / dW shapes (profiles/r01_tf32_mode.md).
bool wide_pair_enabled() { return pair_enabled() && g_tc_terms == 3; }

// output tiles of a launch: 128-row tiles, or 256-row pair tiles
int nt_tiles(const GemmGroup& p, int bn, bool pair) {
  const int bm = tc::BM * (pair ? 2 : 1);
  int t = 0;
  for (int j = 0; j < p.njobs; ++j) t += ((p.rows + bm - 1) / bm) * ((p.job[j].n + bn - 1) / bn);
  return t;
}

int nt_min_stages(const GemmGroup& p) {
  int kst = 1 << 30;
  for (int j = 0; j < p.njobs; ++j) {
    int st = 0;
    for (int s = 0; s < p.job[j].nseg; ++s) st += (p.job[j].seg[s].k + kTmaNtBk - 1) / kTmaNtBk;
    kst = st < kst ? st : kst;
  }
  return kst;
}

bool csplit_enabled();

struct NtConfig {
  int bn = 32, splits = 1;
  bool pair = false;
};

// Tile shape of a launch.  TMA launches prefer CTA pairs (256 x BN tiles,
// half of B per CTA); when there are too few tiles to cover the SMs and K is
// deep, the K range is split over up to 4 tiles' worth of blocks (narrow
// tiles instead re-read and re-convert A once per tile column).
NtConfig nt_config(const GemmGroup& p) {
  NtConfig c;
  c.bn = tc::pick_bn([&](int b) { return nt_tiles(p, b, false); });
  static int split_env = -2;  // RGB_TC_SPLIT=0 disables split-K (tuning experiments)
  if (split_env == -2) {
    const char* e = getenv("RGB_TC_SPLIT");
    split_env = e ? atoi(e) : -1;
  }
  if (!p.tma || getenv("RGB_TC_BN")) return c;
  const int kst = nt_min_stages(p);
  auto split_for = [&](int ctas) {
    int sp = 148 / (ctas > 0 ? ctas : 1);
    sp = sp > 4 ? 4 : sp;
    while (sp > 1 && kst / sp < 8) --sp;  // at least 8 K-stages per split
    return split_env == 0 ? 1 : (sp < 1 ? 1 : sp);
  };
  if (pair_enabled()) {
    // pairs only when they fill the machine without split-K: small (per-frame)
    // products with a short K range lose more to the pair's longer pipeline
    // start than they gain (cfg4 per-frame GEMMs: 5.2 -> 6.0 ms per step)
    static int pair_bn = -1;  // RGB_TC_PAIR_BN: force 256 / 128 (tuning experiments)
    if (pair_bn < 0) {
      const char* e = getenv("RGB_TC_PAIR_BN");
      pair_bn = e ? atoi(e) : 0;
    }
    for (int bn : {256, 128}) {
      if (pair_bn && bn != pair_bn) continue;
      if (wide_pair_enabled() && 2 * nt_tiles(p, bn, true) >= 120) {
        c.bn = bn;
        c.pair = true;
        return c;
      }
    }
    // few pair tiles, deep K: CTA pairs with cluster split-K (the splits of a
    // pair tile form one cluster of 2*splits CTAs and reduce through DSMEM)
    // (opt-in, RGB_TC_PAIRSPLIT=1: measured 2x slower than unpaired split-K on
    // the cfg4 per-frame shapes -- 8-CTA clusters of ~200 KB CTAs do not all
    // fit at once -- kept for other shapes / future tuning)
    static int pair_split = -1;
    if (pair_split < 0) {
      const char* e = getenv("RGB_TC_PAIRSPLIT");
      pair_split = e ? atoi(e) != 0 : 0;
    }
    if (pair_split && csplit_enabled() && split_env != 0) {
      for (int bn : {256, 128}) {
        if (pair_bn && bn != pair_bn) continue;
        const int ctas = 2 * nt_tiles(p, bn, true);
        const int sp = split_for(ctas);
        if (sp > 1 && ctas * sp >= 96) {
          c.bn = bn;
          c.pair = true;
          c.splits = sp;
          return c;
        }
      }
    }
  }
  if (c.bn >= 128) return c;
  const int sp = split_for(nt_tiles(p, 128, false));
  if (sp > 1) {
    c.bn = 128;
    c.splits = sp;
  }
  return c;
}

long long nt_scratch(const GemmGroup& p, const NtConfig& c) {
  return c.splits > 1 ? (long long)nt_tiles(p, c.bn, c.pair) * (c.pair ? 2 : 1) * c.splits * tc::BM * c.bn : 0;
}

bool persist_enabled() {  // RGB_TC_PERSIST=0 disables the persistent kernels (tuning experiments); rgb_set_tc_config overrides
  int& on = g_tc_opt[1];
  if (on < 0) {
    const char* e = getenv("RGB_TC_PERSIST");
    on = e ? atoi(e) != 0 : 1;
  }
  return on == 1;
}

// persistent kernel for launches of at least two waves, or of deep K
bool use_persistent(int blocks, int bn, int stages_per_acc = 0) {
  return (persist_enabled() && blocks > 148 && bn >= 128) || stages_per_acc > tc::kMaxStagesPerAcc;
}

template <bool PAIR>
void launch_nt_bn(const GemmGroup& p, int bn, int blocks, cudaStream_t s, int cluster = 1) {
  if (bn == 256) tc::launch_tma<256, false, PAIR>(p, blocks, s, cluster);
  else if (bn == 128) tc::launch_tma<128, false, PAIR>(p, blocks, s, cluster);
  else if constexpr (!PAIR) {
    if (bn == 64) tc::launch_tma<64, false, false>(p, blocks, s, cluster);
    else tc::launch_tma<32, false, false>(p, blocks, s, cluster);
  }
}

bool csplit_enabled() {  // RGB_TC_CSPLIT=0: split-K through global partials + fixup kernel (experiments); rgb_set_tc_config overrides
  int& on = g_tc_opt[2];
  if (on < 0) {
    const char* e = getenv("RGB_TC_CSPLIT");
    on = e ? atoi(e) != 0 : 1;
  }
  return on == 1;
}

}  // namespace

long long tc_gemm_nt_scratch(const GemmGroup& p) {
  const NtConfig c = nt_config(p);
  return csplit_enabled() && !c.pair ? 0 : nt_scratch(p, c);
}

int nt_max_stages(const GemmGroup& p) {
  int kst = 0;
  for (int j = 0; j < p.njobs; ++j) {
    int st = 0;
    for (int s = 0; s < p.job[j].nseg; ++s) st += (p.job[j].seg[s].k + kTmaNtBk - 1) / kTmaNtBk;
    kst = st > kst ? st : kst;
  }
  return kst;
}

// tile width of K-chunked CTA-pair launches: 256 (half of B per CTA; one
// chunk accumulator beside R) measured 1.3x faster at the cfg4 shapes than 128
// (three chunk accumulators, but twice the A traffic per FLOP); RGB_TC_CHUNK_BN
// overrides
int chunk_pair_bn() {
  static int bn = -1;
  if (bn < 0) {
    const char* e = getenv("RGB_TC_CHUNK_BN");
    bn = e ? atoi(e) : 256;
  }
  return bn == 128 ? 128 : 256;
}

int launch_tc_gemm_nt(GemmGroup p, cudaStream_t s) {
  p.terms = g_tc_terms;
  NtConfig c = nt_config(p);
  // deep K without split-K: the K-chunked persistent kernel (accuracy)
  const int acc_stages = (nt_max_stages(p) * (p.terms == 1 ? 1 : 3) + 2) / 3 / std::max(c.splits, 1);
  if (p.tma && acc_stages > tc::kMaxStagesPerAcc) {
    if (c.bn < 128) c.bn = 128;
    if (c.pair) c.bn = chunk_pair_bn();
    c.splits = 1;
  }
  p.csplit = c.splits > 1 && csplit_enabled() ? 1 : 0;
  if (c.pair && c.splits > 1 && !p.csplit) c.splits = 1;  // pairs split only through the cluster
  if (c.splits > 1 && !p.csplit && (!p.part || nt_scratch(p, c) > p.part_cap)) c.splits = 1;  // no scratch
  if (!p.tma) c = NtConfig{tc::pick_bn([&](int b) { return nt_tiles(p, b, false); }), 1, false};
  p.splits = c.splits;
  p.pair = c.pair ? 1 : 0;
  const int bm = tc::BM * (c.pair ? 2 : 1);
  p.tile_start[0] = 0;
  for (int j = 0; j < p.njobs; ++j) {
    p.tiles_n[j] = (p.job[j].n + c.bn - 1) / c.bn;
    p.tile_start[j + 1] = p.tile_start[j] + ((p.rows + bm - 1) / bm) * p.tiles_n[j];
  }
  const int blocks = p.tile_start[p.njobs] * c.splits * (c.pair ? 2 : 1);
  if (blocks == 0) return 0;
  static const bool log = getenv("RGB_TC_LOG") != nullptr;  // shape log (tuning)
  if (log) {
    fprintf(stderr, "[tc nt] rows %d jobs %d n0 %d kst %d nseg %d epi_ops %d bn %d pair %d splits %d tiles %d blocks %d persistent %d\n",
            p.rows, p.njobs, p.job[0].n, nt_max_stages(p), p.job[0].nseg, p.job[0].epi.nops, c.bn, (int)c.pair,
            c.splits, p.tile_start[p.njobs], blocks, (int)(p.tma && c.splits == 1 && use_persistent(blocks, c.bn, acc_stages)));
  }
  if (p.tma && c.splits == 1 && use_persistent(blocks, c.bn, acc_stages)) {
    const int ntiles = p.tile_start[p.njobs];
    if (c.pair) {
      if (c.bn == 256) tc::launch_persistent<256, false, true>(p, ntiles, nt_max_stages(p), s);
      else tc::launch_persistent<128, false, true>(p, ntiles, nt_max_stages(p), s);
    } else {
      if (c.bn == 256) tc::launch_persistent<256, false, false>(p, ntiles, nt_max_stages(p), s);
      else tc::launch_persistent<128, false, false>(p, ntiles, nt_max_stages(p), s);
    }
  } else if (p.tma) {
    if (c.pair) launch_nt_bn<true>(p, c.bn, blocks, s, p.csplit ? c.splits : 1);
    else launch_nt_bn<false>(p, c.bn, blocks, s, p.csplit ? c.splits : 1);
  } else {
    if (c.bn == 256) tc::launch_one<256, false>(p, blocks, s);
    else if (c.bn == 128) tc::launch_one<128, false>(p, blocks, s);
    else if (c.bn == 64) tc::launch_one<64, false>(p, blocks, s);
    else tc::launch_one<32, false>(p, blocks, s);
  }
  if (c.splits == 1 || p.csplit) return 1;
  int64_t maxq = 0;
  for (int j = 0; j < p.njobs; ++j) maxq = std::max<int64_t>(maxq, (int64_t)p.rows * p.job[j].n);
  maxq = (maxq + 3) / 4;
  int eblocks = (int)std::min<int64_t>((maxq + 255) / 256, 148 * 8);
  eblocks = eblocks < 1 ? 1 : eblocks;
  if (c.bn == 256) tc::splitk_epilogue_kernel<256><<<dim3(eblocks, p.njobs), 256, 0, s>>>(p);
  else tc::splitk_epilogue_kernel<128><<<dim3(eblocks, p.njobs), 256, 0, s>>>(p);
  return 2;
}


// Persistent frame loop (tma_frame_loop_kernel): -1 when the loop's GEMM step
// does not suit it (the caller then launches per frame), else a CUDA status.
// The jobs must share their A segments and width (tiles span every job);
// the tile width per job (bu) and the K split are chosen so that 96..148 CTAs
// run, preferring no split (no DSMEM reduction).  fuse_ew: the elementwise
// steps are element-local over the jobs' width and run in the epilogue.
int launch_tc_frame_loop(const GemmGroup& g0, const GemmGroup* d_frames, const EwLaunch* d_ew, int n_ew,
                         int fuse_ew, int pattern, const EwLaunch* d_tail, int nframes, unsigned* bar,
                         cudaStream_t s) {
  GemmGroup p = g0;
  p.terms = g_tc_terms;
  if (!p.tma || p.njobs < 1 || p.njobs > 4) return -1;
  const int W = p.job[0].n, J = p.njobs;
  for (int j = 1; j < J; ++j) {
    if (p.job[j].n != W || p.job[j].nseg != p.job[0].nseg) return -1;
    for (int q = 0; q < p.job[0].nseg; ++q)
      if (p.job[j].seg[q].a != p.job[0].seg[q].a || p.job[j].seg[q].k != p.job[0].seg[q].k) return -1;
  }
  const int mt = (p.rows + tc::BM - 1) / tc::BM;
  static int forced_bu = -1, forced_split = -1;  // RGB_FL_BU / RGB_FL_SPLIT: experiments
  if (forced_bu < 0) {
    const char* e = getenv("RGB_FL_BU");
    forced_bu = e ? atoi(e) : 0;
    e = getenv("RGB_FL_SPLIT");
    forced_split = e ? atoi(e) : 0;
  }
  // Tile width first: the main loop is bound by L2 -> SM operand traffic
  // (A is re-read once per unit block, B once per 128-row block), so the
  // widest tile (J * bu = 128) wins, then the smallest K split that still
  // occupies >= 96 SMs (tools/trace_frame_loop.py, cfg4: forward J=2 bu=64
  // split 2, backward J=1 bu=128 split 4; bu=32 without a split was 1.7x
  // slower in the main loop).
  int bu = 0, sp = 1;
  for (int cand : {128, 64, 32}) {
    if (forced_bu && cand != forced_bu) continue;
    if (J * cand > 128 || J * cand < 32) continue;
    for (int split : {1, 2, 4}) {
      if (forced_split && split != forced_split) continue;
      const int ctas = mt * ((W + cand - 1) / cand) * split;
      if (ctas >= (forced_bu || forced_split ? 1 : 96) && ctas <= 148) {
        bu = cand;
        sp = split;
        break;
      }
    }
    if (bu) break;
  }
  if (!bu || (sp > 1 && !csplit_enabled())) return -1;
  const int BN = J * bu;
  p.splits = sp;
  p.csplit = sp > 1 ? 1 : 0;
  p.pair = 0;
  const int blocks = mt * ((W + bu - 1) / bu) * sp;
  static int prefetch = -1;  // RGB_FL_PREFETCH=0: no L2 prefetch of the chains' operands (experiments)
  if (prefetch < 0) {
    const char* e = getenv("RGB_FL_PREFETCH");
    prefetch = e ? atoi(e) != 0 : 0;  // off: 1 measured 554k -> 418k frames/s (the bulk prefetches delay the TMA loads)
  }
  static int fwd = -1;  // RGB_FL_FORWARD=0: chains through global memory (experiments)
  if (fwd < 0) {
    const char* e = getenv("RGB_FL_FORWARD");
    fwd = e ? atoi(e) != 0 : 0;  // off: the register-forwarding evaluator spills (168-register cap) and measured slower
  }
  static int pat_env = -1;  // RGB_FL_PATTERN=0: the generic chain evaluator (experiments)
  if (pat_env < 0) {
    const char* e = getenv("RGB_FL_PATTERN");
    pat_env = e ? atoi(e) != 0 : 1;
  }
  if (!pat_env || (pattern == 1 && !(J == 2 && bu % 4 == 0)) || (pattern == 2 && J != 1)) pattern = 0;
  // RGB_FL_PRELOAD: 0 the pattern's operands are loaded after the reduction,
  // 1 preloaded by the store warps (forward and backward), 2 forward only
  static int preload_env = -1;
  if (preload_env < 0) {
    const char* e = getenv("RGB_FL_PRELOAD");
    preload_env = e ? atoi(e) : 1;
  }
  const int preload = preload_env == 1 || (preload_env == 2 && pattern == 1);
  tc::FrameLoop fl{d_frames, d_ew, nframes, n_ew, fuse_ew, bu, prefetch, fwd, pattern, preload,
                   pattern ? d_tail : nullptr, bar};
  auto launch = [&](auto kernel, int smem) -> int {
    static bool bad = false;  // cooperative cluster launches unsupported: stay per-frame
    if (bad) return -1;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(tc::kFrameThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = sp;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = sp > 1 ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, fl, p);
    if (e == cudaErrorInvalidValue || e == cudaErrorNotSupported || e == cudaErrorCooperativeLaunchTooLarge) {
      cudaGetLastError();
      bad = e != cudaErrorCooperativeLaunchTooLarge;
      return -1;
    }
    return (int)e;
  };
  if (BN == 128) return launch(tc::tma_frame_loop_kernel<128>, tc::FCfg<128>::SMEM);
  if (BN == 64) return launch(tc::tma_frame_loop_kernel<64>, tc::FCfg<64>::SMEM);
  if (BN == 32) return launch(tc::tma_frame_loop_kernel<32>, tc::FCfg<32>::SMEM);
  if (BN == 96) return launch(tc::tma_frame_loop_kernel<96>, tc::FCfg<96>::SMEM);
  return -1;
}

void launch_tc_gemm_dw(DwGroup p, cudaStream_t s) {
  p.terms = g_tc_terms;
  const bool pair = p.tma && wide_pair_enabled() && !getenv("RGB_TC_BN");
  const int bm = tc::BM * (pair ? 2 : 1);
  auto tiles_for = [&](int bn) {
    int t = 0;
    for (int j = 0; j < p.njobs; ++j) t += ((p.job[j].m + bm - 1) / bm) * ((p.job[j].n + bn - 1) / bn);
    return t * (pair ? 2 : 1);
  };
  int bn = tc::pick_bn(tiles_for);
  if (pair && bn < 128) bn = 128;
  // deep K (the window rows h*S): the K-chunked persistent kernel (accuracy)
  const int acc_stages = ((p.k + 31) / 32 * (p.terms == 1 ? 1 : 3) + 2) / 3;
  if (p.tma && acc_stages > tc::kMaxStagesPerAcc) bn = pair ? chunk_pair_bn() : std::max(bn, 128);
  p.tile_start[0] = 0;
  for (int j = 0; j < p.njobs; ++j) {
    p.tiles_n[j] = (p.job[j].n + bn - 1) / bn;
    p.tile_start[j + 1] = p.tile_start[j] + ((p.job[j].m + bm - 1) / bm) * p.tiles_n[j];
  }
  const int blocks = p.tile_start[p.njobs] * (pair ? 2 : 1);
  if (blocks == 0) return;
  if (p.tma && use_persistent(blocks, bn, acc_stages)) {
    const int ntiles = p.tile_start[p.njobs];
    if (pair) {
      if (bn == 256) tc::launch_persistent<256, true, true>(p, ntiles, (p.k + 31) / 32, s);
      else tc::launch_persistent<128, true, true>(p, ntiles, (p.k + 31) / 32, s);
    } else {
      if (bn == 256) tc::launch_persistent<256, true, false>(p, ntiles, (p.k + 31) / 32, s);
      else tc::launch_persistent<128, true, false>(p, ntiles, (p.k + 31) / 32, s);
    }
  } else if (p.tma) {
    if (pair) {
      if (bn == 256) tc::launch_tma<256, true, true>(p, blocks, s);
      else tc::launch_tma<128, true, true>(p, blocks, s);
    } else {
      if (bn == 256) tc::launch_tma<256, true, false>(p, blocks, s);
      else if (bn == 128) tc::launch_tma<128, true, false>(p, blocks, s);
      else if (bn == 64) tc::launch_tma<64, true, false>(p, blocks, s);
      else tc::launch_tma<32, true, false>(p, blocks, s);
    }
  } else {
    if (bn == 256) tc::launch_one<256, true>(p, blocks, s);
    else if (bn == 128) tc::launch_one<128, true>(p, blocks, s);
    else if (bn == 64) tc::launch_one<64, true>(p, blocks, s);
    else tc::launch_one<32, true>(p, blocks, s);
  }
}

}  // namespace rgb

namespace rgb {
void set_tc_terms(int terms) { g_tc_terms = terms; }
int get_tc_terms() { return g_tc_terms; }
void set_tc_config(int pair, int persist, int csplit) {
  if (pair >= 0) g_tc_opt[0] = pair != 0;
  if (persist >= 0) g_tc_opt[1] = persist != 0;
  if (csplit >= 0) g_tc_opt[2] = csplit != 0;
}
}  // namespace rgb

#ifdef RGB_FL_TRACE
extern "C" int rgb_exp_fl_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, rgb::tc::g_fl_trace, sizeof(rgb::tc::g_fl_trace)) == cudaSuccess ? 0 : 3;  // [64][16]
}
#endif
#ifdef RGB_EXP_TRACE
extern "C" int rgb_exp_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, rgb::tc::g_trace, sizeof(rgb::tc::g_trace)) == cudaSuccess ? 0 : 3;  // [6][1024]
}
extern "C" int rgb_exp_cta(long long* out) {
  return cudaMemcpyFromSymbol(out, rgb::tc::g_cta, sizeof(rgb::tc::g_cta)) == cudaSuccess ? 0 : 3;
}
#endif
