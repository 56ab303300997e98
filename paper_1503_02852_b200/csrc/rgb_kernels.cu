// SIMT fp32 kernels of the graph-RNN step.  See rgb_kernels.cuh for the list.
// Reference semantics cited per function (/root/reference/pkg/src/rnngraph/).
#include "rgb_kernels.cuh"
#include "rgb_ew.cuh"

#include <cmath>
#include <cstdlib>

namespace rgb {

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ew_chain_kernel(const __grid_constant__ EwLaunch p) {
  // chain staged in shared memory: per-element indexed reads of the parameter
  // block miss the constant cache (see rgb_tc_gemm.cu kChainBytes)
  __shared__ __align__(16) int chain_words[sizeof(EwChain) / 4];
  const int* src = reinterpret_cast<const int*>(&p.chain[blockIdx.y]);
  for (int i = threadIdx.x; i < (int)(sizeof(EwChain) / 4); i += blockDim.x) chain_words[i] = src[i];
  __syncthreads();
  const EwChain& ch = *reinterpret_cast<const EwChain*>(chain_words);
  pdl_wait();  // predecessor complete (PDL launches inside frame loops)
  pdl_trigger();
  if (chain_vec_ok(ch, ch.width)) {
    // 16-byte path: one thread per 4 consecutive units of a row
    const int w4 = ch.width / 4;
    const int64_t nq = (int64_t)p.rows * w4;
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    // 32-bit index arithmetic (a 64-bit division is a long subroutine call)
    if (nq >= (int64_t)UINT32_MAX) __trap();
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < (uint32_t)nq; q += gridDim.x * blockDim.x) {
      const uint32_t r32 = q / (uint32_t)w4;
      const int64_t rr[1] = {(int64_t)r32};
      const int j = (int)(q - r32 * (uint32_t)w4) * 4;
      const bool ok[1] = {true};
      const float4 acc[1] = {zero};
      ew_chain_vec<1>(ch, ch.width, rr, j, ok, p.ring, false, acc);
    }
    return;
  }
  const int64_t total = (int64_t)p.rows * ch.width;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ch.width;
    const int j = (int)(e - r * ch.width);
    for (int k = 0; k < ch.nops; ++k) ew_apply(ch.op[k], ch.width, r, j, p.ring, false, 0.0f);
  }
}

namespace {
bool g_pdl_scope = false;
}

void set_pdl_scope(bool on) { g_pdl_scope = on; }

bool pdl_active() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("RGB_PDL");
    env = e ? atoi(e) != 0 : 1;
  }
  return env == 1 && g_pdl_scope;
}

void launch_ew(const EwLaunch& p, cudaStream_t s) {
  int64_t maxw = 1;
  for (int c = 0; c < p.nchains; ++c) maxw = maxw > p.chain[c].width ? maxw : p.chain[c].width;
  int64_t total = (int64_t)p.rows * maxw;
  if (maxw % 4 == 0) total /= 4;  // the 16-byte path: one thread per 4 units
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  if (pdl_active()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks, p.nchains);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, ew_chain_kernel, p);
  } else {
    ew_chain_kernel<<<dim3(blocks, p.nchains), 256, 0, s>>>(p);
  }
}

// ---------------------------------------------------------------------------
// grouped NT GEMM: C[r, n] = sum_seg sum_k A[r, k] * B[n, k], epilogue = EW chain
// (the per-edge products of _accum_z / backward_layer, engine.py:304-321, 525-535)

constexpr int BM = 64, BN = 64, BK = 16;

__device__ __forceinline__ void find_job(const int* tile_start, int njobs, int bid, int& job, int& tile) {
  job = 0;
  while (job + 1 < njobs && bid >= tile_start[job + 1]) ++job;
  tile = bid - tile_start[job];
}

__global__ void __launch_bounds__(256) gemm_nt_kernel(const __grid_constant__ GemmGroup p) {
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  __shared__ __align__(16) int chain_words[sizeof(EwChain) / 4];
  int jid, tile;
  find_job(p.tile_start, p.njobs, blockIdx.x, jid, tile);
  const GemmJob& job = p.job[jid];
  {
    const int* src = reinterpret_cast<const int*>(&job.epi);
    for (int i = threadIdx.x; i < (int)(sizeof(EwChain) / 4); i += blockDim.x) chain_words[i] = src[i];
  }
  const EwChain& epi = *reinterpret_cast<const EwChain*>(chain_words);
  const RingWrite ring = p.ring;
  const int tm = tile / p.tiles_n[jid], tn = tile % p.tiles_n[jid];
  const int m0 = tm * BM, n0 = tn * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  const int lrow = threadIdx.x / 4, lk = (threadIdx.x % 4) * 4;
  for (int s = 0; s < job.nseg; ++s) {
    const Seg sg = job.seg[s];
    for (int k0 = 0; k0 < sg.k; k0 += BK) {
      {
        const int gr = m0 + lrow;
        #pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int gk = k0 + lk + i;
          As[lk + i][lrow] = (gr < p.rows && gk < sg.k) ? sg.a[(int64_t)gr * sg.k + gk] : 0.0f;
        }
        const int gn = n0 + lrow;
        #pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int gk = k0 + lk + i;
          Bs[lk + i][lrow] = (gn < job.n && gk < sg.k) ? sg.b[(int64_t)gn * sg.k + gk] : 0.0f;
        }
      }
      __syncthreads();
      #pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        #pragma unroll
        for (int i = 0; i < 4; ++i)
          #pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  #pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
    if (r >= p.rows) continue;
    #pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c >= job.n) continue;
      for (int k = 0; k < epi.nops; ++k) ew_apply(epi.op[k], job.n, r, c, ring, k == 0, acc[i][j]);
    }
  }
}

void launch_gemm_nt(const GemmGroup& p, cudaStream_t s) {
  const int tiles = p.tile_start[p.njobs];
  if (tiles > 0) gemm_nt_kernel<<<tiles, 256, 0, s>>>(p);
}

// ---------------------------------------------------------------------------
// dW: G[m, n] = alpha * sum_k E[k, m] * Y[k, n]   (engine.py:578-599, paper Eq. 19)

__global__ void __launch_bounds__(256) gemm_dw_kernel(const __grid_constant__ DwGroup p) {
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  int jid, tile;
  find_job(p.tile_start, p.njobs, blockIdx.x, jid, tile);
  const DwJob& job = p.job[jid];
  const int tm = tile / p.tiles_n[jid], tn = tile % p.tiles_n[jid];
  const int m0 = tm * BM, n0 = tn * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  const int lk = threadIdx.x / 16, lc = (threadIdx.x % 16) * 4;  // 16 k-rows x 64 columns
  for (int k0 = 0; k0 < p.k; k0 += BK) {
    const int gk = k0 + lk;
    #pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gm = m0 + lc + i, gn = n0 + lc + i;
      As[lk][lc + i] = (gk < p.k && gm < job.m) ? job.e[(int64_t)gk * job.m + gm] : 0.0f;
      Bs[lk][lc + i] = (gk < p.k && gn < job.n) ? job.y[(int64_t)gk * job.n + gn] : 0.0f;
    }
    __syncthreads();
    #pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
      #pragma unroll
      for (int i = 0; i < 4; ++i)
        #pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  #pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= job.m) continue;
    #pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < job.n) job.g[(int64_t)m * job.n + n] = p.alpha * acc[i][j];
    }
  }
}

void launch_gemm_dw(const DwGroup& p, cudaStream_t s) {
  const int tiles = p.tile_start[p.njobs];
  if (tiles > 0) gemm_dw_kernel<<<tiles, 256, 0, s>>>(p);
}

// ---------------------------------------------------------------------------
// Narrow dW (n <= 4, e.g. the bias edge from the constant-one layer):
// G[m, j] = alpha * sum_r E[r, m] * Y[r, j].  A tensor-core tile would be
// 97% padding; this is a GEMV-shaped HBM stream of E instead.  Pass 1: block
// (job, 128-unit group, K chunk), lane = 4 consecutive units (16-byte loads),
// warp w takes rows w, w+8, ...; warps reduced in fixed order into part[].
// Pass 2 sums the chunks in order: bitwise reproducible.
constexpr int kNarrowChunk = 1024;  // rows per K chunk

__device__ __forceinline__ void narrow_locate(const DwGroup& p, int b, int nchunks, int& job, int& grp, int& chunk) {
  job = 0;
  int base = 0;
  for (;;) {
    const int groups = (p.job[job].m + 127) / 128;
    if (b < base + groups * nchunks || job + 1 == p.njobs) break;
    base += groups * nchunks;
    ++job;
  }
  const int local = b - base;
  grp = local / nchunks;
  chunk = local % nchunks;
}

__global__ void __launch_bounds__(256) dw_narrow_kernel(const __grid_constant__ DwGroup p, float* part,
                                                        int nchunks) {
  __shared__ float red[8][128][4];
  int job, grp, chunk;
  narrow_locate(p, blockIdx.x, nchunks, job, grp, chunk);
  const DwJob& jb = p.job[job];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m = jb.m, n = jb.n;
  const int u0 = grp * 128 + lane * 4;
  const int r0 = chunk * kNarrowChunk, r1 = min(p.k, r0 + kNarrowChunk);
  float acc[4][4] = {};
  for (int r = r0 + warp; r < r1; r += 8) {
    float e[4];
    if (u0 + 3 < m && (m & 3) == 0) {
      const float4 v = *reinterpret_cast<const float4*>(jb.e + (int64_t)r * m + u0);
      e[0] = v.x, e[1] = v.y, e[2] = v.z, e[3] = v.w;
    } else {
      for (int t = 0; t < 4; ++t) e[t] = u0 + t < m ? jb.e[(int64_t)r * m + u0 + t] : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= n) break;
      const float y = jb.y[(int64_t)r * n + j];
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[j][t] = fmaf(e[t], y, acc[j][t]);
    }
  }
  for (int t = 0; t < 4; ++t)
    for (int j = 0; j < 4; ++j) red[warp][lane * 4 + t][j] = acc[j][t];
  __syncthreads();
  // fixed-order reduction over the 8 warps; thread = (unit, j)
  for (int q = threadIdx.x; q < 128 * 4; q += 256) {
    const int u = q / 4, j = q % 4;
    if (j >= n || grp * 128 + u >= m) continue;
    float s = 0.0f;
    for (int w = 0; w < 8; ++w) s += red[w][u][j];
    part[((size_t)blockIdx.x) * 512 + q] = s;
  }
}

__global__ void __launch_bounds__(256) dw_narrow_sum_kernel(const __grid_constant__ DwGroup p, const float* part,
                                                            int nchunks) {
  // one thread per (job, unit, j); blocks of pass 1 are laid out job-major,
  // then unit group, then chunk
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  int base_blocks = 0;
  for (int job = 0; job < p.njobs; ++job) {
    const DwJob& jb = p.job[job];
    const int groups = (jb.m + 127) / 128;
    const int cnt = jb.m * jb.n;
    if (q < cnt) {
      const int u = q / jb.n, j = q % jb.n;
      const int grp = u / 128, ul = u % 128;
      const float* src = part + ((size_t)(base_blocks + grp * nchunks)) * 512 + ul * 4 + j;
      float s = 0.0f;
      for (int c = 0; c < nchunks; ++c) s += src[(size_t)c * 512];
      jb.g[(int64_t)u * jb.n + j] = p.alpha * s;
      return;
    }
    q -= cnt;
    base_blocks += groups * nchunks;
  }
}

long long dw_narrow_scratch(const DwGroup& p) {
  const int nchunks = (p.k + kNarrowChunk - 1) / kNarrowChunk;
  long long blocks = 0;
  for (int j = 0; j < p.njobs; ++j) blocks += (long long)((p.job[j].m + 127) / 128) * nchunks;
  return blocks * 512;
}

int launch_dw_narrow(const DwGroup& p, float* part, cudaStream_t s) {
  const int nchunks = (p.k + kNarrowChunk - 1) / kNarrowChunk;
  int blocks = 0, outs = 0;
  for (int j = 0; j < p.njobs; ++j) {
    blocks += ((p.job[j].m + 127) / 128) * nchunks;
    outs += p.job[j].m * p.job[j].n;
  }
  if (blocks == 0) return 0;
  dw_narrow_kernel<<<blocks, 256, 0, s>>>(p, part, nchunks);
  dw_narrow_sum_kernel<<<(outs + 255) / 256, 256, 0, s>>>(p, part, nchunks);
  return 2;
}

// ---------------------------------------------------------------------------
// softmax over each row, max-subtracted (kernels.py:159-173); one warp per row

__global__ void softmax_rows_kernel(float* y, int rows, int width, RingWrite ring, int is_ring) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  float* row = y + (int64_t)warp * width;
  float m = -INFINITY;
  for (int j = lane; j < width; j += 32) m = fmaxf(m, row[j]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.0f;
  for (int j = lane; j < width; j += 32) s += expf(row[j] - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = 1.0f / s;
  for (int j = lane; j < width; j += 32) {
    const float v = expf(row[j] - m) * inv;
    ring_store(y, (int64_t)warp * width + j, warp, width, is_ring != 0, ring, v);
  }
}

void launch_softmax(float* y, int rows, int width, RingWrite ring, bool is_ring, cudaStream_t s) {
  const int threads = 256, per = threads / 32;
  softmax_rows_kernel<<<(rows + per - 1) / per, threads, 0, s>>>(y, rows, width, ring, is_ring ? 1 : 0);
}

// ---------------------------------------------------------------------------
// delta_out = d - y and the per-row loss (engine.py:425-474)

__global__ void inject_loss_kernel(const float* y, const void* target, int target_kind, int criterion, float* inj,
                                   double* row_loss, int rows, int width, int* bad) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float* yr = y + (int64_t)warp * width;
  float* ir = inj + (int64_t)warp * width;
  double loss = 0.0;
  if (target_kind == 2) {
    const float* dr = static_cast<const float*>(target) + (int64_t)warp * width;
    for (int j = lane; j < width; j += 32) {
      const float d = dr[j], v = yr[j];
      ir[j] = d - v;
      if (criterion == 1) {
        const double diff = (double)d - (double)v;
        loss += 0.5 * diff * diff;
      } else if (d != 0.0f) {
        loss -= (double)d * log((double)v);
      }
    }
  } else {
    const long long id = target_kind == 0 ? static_cast<const long long*>(target)[warp]
                                          : (long long)static_cast<const int*>(target)[warp];
    for (int j = lane; j < width; j += 32) ir[j] = (j == id ? 1.0f : 0.0f) - yr[j];
    if (lane == 0) {
      if (id >= 0 && id < width) {
        loss = -log((double)yr[id]);
      } else {  // the reference raises IndexError (engine.py:443-456): poison the loss, flag the plan
        loss = __longlong_as_double(0x7ff8000000000000LL);
        if (bad) atomicOr(bad, 2);
      }
    }
  }
  for (int o = 16; o; o >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, o);
  if (lane == 0) row_loss[warp] = loss;
}

void launch_inject_loss(const float* y, const void* target, int target_kind, int criterion, float* inj,
                        double* row_loss, int rows, int width, int* bad, cudaStream_t s) {
  const int threads = 256, per = threads / 32;
  inject_loss_kernel<<<(rows + per - 1) / per, threads, 0, s>>>(y, target, target_kind, criterion, inj, row_loss,
                                                                rows, width, bad);
}

// fixed-order fp64 sum (deterministic run to run)
__global__ void sum_rows_kernel(const double* v, int n, double* out) {
  __shared__ double part[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) s += v[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

void launch_sum_rows(const double* row_loss, int rows, double* out, cudaStream_t s) {
  sum_rows_kernel<<<1, 256, 0, s>>>(row_loss, rows, out);
}

// ---------------------------------------------------------------------------
// SGD fused with the W^T refresh (engine.py:606-612, 138-139): per 32x32 tile
// of every dense connection, W -= lr * G in place and the updated tile is
// written transposed into W^T -- one pass (8 B read + 8 B written per
// parameter instead of a separate update and transpose pass).
__global__ void transpose_kernel(const __grid_constant__ TransposeGroup p) {
  __shared__ float t[32][33];
  int jid, tile;
  find_job(p.tile_start, p.njobs, blockIdx.x, jid, tile);
  const TransposeJob& jb = p.job[jid];
  const int r0 = (tile / p.tiles_c[jid]) * 32, c0 = (tile % p.tiles_c[jid]) * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + tx;
    if (r < jb.rows && c < jb.cols) {
      const int64_t e = (int64_t)r * jb.cols + c;
      float v = jb.src[e];
      if (jb.g) {
        v -= p.lr * jb.g[e];
        jb.src[e] = v;
      }
      t[i][tx] = v;
    }
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + tx;
    if (r < jb.rows && c < jb.cols) jb.dst[(int64_t)c * jb.rows + r] = t[tx][i];
  }
}

void launch_transpose(const TransposeGroup& p, cudaStream_t s) {
  const int tiles = p.tile_start[p.njobs];
  if (tiles > 0) transpose_kernel<<<tiles, 256, 0, s>>>(p);
}

__global__ void fill_kernel(float* p, float v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

void launch_fill(float* p, float v, int64_t n, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  fill_kernel<<<(int)blocks, 256, 0, s>>>(p, v, n);
}

// token ids -> one-hot rows; id < 0 means "before the stream started": a zero
// row (kernels.py:106-115 semantics of rows_gather_add)
__global__ void onehot_kernel(const int64_t* ids, int rows, int width, float* out) {
  const int64_t total = (int64_t)rows * width;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / width;
    out[e] = (ids[r] == e - r * width) ? 1.0f : 0.0f;
  }
}

void launch_onehot(const int64_t* ids, int rows, int width, float* out, cudaStream_t s) {
  int64_t blocks = ((int64_t)rows * width + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  onehot_kernel<<<(int)blocks, 256, 0, s>>>(ids, rows, width, out);
}

__global__ void count_nonfinite_kernel(const float* p, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += isfinite(p[i]) ? 0ull : 1ull;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

void launch_count_nonfinite(const float* p, int64_t n, unsigned long long* out, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  count_nonfinite_kernel<<<(int)blocks, 256, 0, s>>>(p, n, out);
}

}  // namespace rgb

// ---------------------------------------------------------------------------
// Token-id input path (reference engine.py:308-316, 588-592; kernels.py:106-140):
// the input layer's history holds ids (int32, -1 = pre-start / reset frame)
// instead of one-hot rows; dense edges out of it gather rows of W^T, their
// gradient is a deterministic scatter over a stable sort of the window rows.
namespace rgb {

__global__ void ids_ring_write_kernel(const int64_t* ids, int32_t* ring, int rows, int S, int64_t t_a, int cap,
                                      int vocab, int* bad) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t t = t_a + r / S;
  const int64_t slot = ((t % cap) + cap) % cap;
  const int n = r % S;
  int32_t v = (int32_t)ids[r];
  if (ids[r] < 0 || ids[r] >= vocab) {  // never gather outside W^T: zero row + plan error flag
    v = -1;
    if (bad) atomicOr(bad, 1);
  }
  ring[slot * S + n] = v;            // the frame's slot
  ring[(slot + cap) * S + n] = v;    // and its mirror
}

void launch_ids_ring_write(const int64_t* ids, int32_t* ring, int rows, int S, int64_t t_a, int cap, int vocab,
                           int* bad, cudaStream_t s) {
  if (rows > 0) ids_ring_write_kernel<<<(rows + 255) / 256, 256, 0, s>>>(ids, ring, rows, S, t_a, cap, vocab, bad);
}

__global__ void ids_reset_kernel(int32_t* ring, int S, int frames, int stream) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < frames) ring[(int64_t)f * S + stream] = -1;
}

void launch_ids_reset(int32_t* ring, int S, int frames, int stream, cudaStream_t s) {
  ids_reset_kernel<<<(frames + 255) / 256, 256, 0, s>>>(ring, S, frames, stream);
}

// out[r, :] (+)= W^T[ids[r], :]  (a zero row for id < 0); W^T is (V x n) row-major
__global__ void gather_rows_kernel(const int32_t* ids, const float* wt, float* out, int rows, int n, int accumulate) {
  const int64_t total = (int64_t)rows * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), j = (int)(e - (int64_t)r * n);
    const int v = ids[r];
    const float g = v >= 0 ? wt[(int64_t)v * n + j] : 0.0f;
    out[e] = accumulate ? out[e] + g : g;
  }
}

void launch_gather_rows(const int32_t* ids, const float* wt, float* out, int rows, int n, bool accumulate,
                        cudaStream_t s) {
  const int64_t total = (int64_t)rows * n;
  int blocks = (int)((total + 255) / 256);
  blocks = blocks > 148 * 16 ? 148 * 16 : (blocks < 1 ? 1 : blocks);
  gather_rows_kernel<<<blocks, 256, 0, s>>>(ids, wt, out, rows, n, accumulate ? 1 : 0);
}

// stable counting sort of the K window rows by id: counts -> offsets -> order
__global__ void id_hist_kernel(const int32_t* ids, int K, int* counts) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < K && ids[r] >= 0) atomicAdd(&counts[ids[r]], 1);  // integer: order-independent
}

// single block: exclusive scan of counts[V] in place (sequential chunks with carry)
__global__ void id_scan_kernel(int* counts, int V) {
  __shared__ int buf[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < V; base += 1024) {
    const int i = base + threadIdx.x;
    const int x = i < V ? counts[i] : 0;
    buf[threadIdx.x] = x;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int y = threadIdx.x >= off ? buf[threadIdx.x - off] : 0;
      __syncthreads();
      buf[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < V) counts[i] = carry + buf[threadIdx.x] - x;  // exclusive
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
}

// one warp walks the rows in order; lanes with equal ids take consecutive
// slots in row order (match_any + rank), so the order is stable and fixed
__global__ void id_place_kernel(const int32_t* ids, int K, int* cursor, int* order) {
  const int lane = threadIdx.x;
  for (int base = 0; base < K; base += 32) {
    const int r = base + lane;
    const int v = r < K ? ids[r] : -2;
    const unsigned same = __match_any_sync(0xffffffffu, v);
    const int rank = __popc(same & ((1u << lane) - 1u));
    const int leader = __ffs(same) - 1;
    int start = 0;
    if (lane == leader && v >= 0) start = cursor[v];
    start = __shfl_sync(0xffffffffu, start, leader);
    if (v >= 0) order[start + rank] = r;
    __syncwarp();
    if (lane == leader && v >= 0) cursor[v] = start + __popc(same);
    __syncwarp();
  }
}

// G[i, v] = alpha * sum over the sorted rows with id v of E[row, i]; one
// thread per unit i walks the sorted rows (coalesced E rows), writing each
// (i, v) once; G must be zero where no row has id v
__global__ void id_scatter_dw_kernel(const float* e, const int32_t* ids, const int* order, int K, int m, int V,
                                     float alpha, float* g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  float acc = 0.0f;
  int cur = -1;
  for (int p = 0; p < K; ++p) {
    const int r = order[p];
    if (r < 0) break;  // fewer valid rows than K (pre-start ids)
    const int v = ids[r];
    if (v != cur) {
      if (cur >= 0) g[(int64_t)i * V + cur] = alpha * acc;
      cur = v;
      acc = 0.0f;
    }
    acc += e[(int64_t)r * m + i];
  }
  if (cur >= 0) g[(int64_t)i * V + cur] = alpha * acc;
}

// scratch: counts[V] + order[K] ints
int launch_id_scatter_dw(const float* e, const int32_t* ids, int K, int m, int V, float alpha, float* g, int* scratch,
                         cudaStream_t s) {
  int* counts = scratch;
  int* order = scratch + V;
  cudaMemsetAsync(counts, 0, (size_t)V * 4, s);
  cudaMemsetAsync(order, 0xff, (size_t)K * 4, s);
  id_hist_kernel<<<(K + 255) / 256, 256, 0, s>>>(ids, K, counts);
  id_scan_kernel<<<1, 1024, 0, s>>>(counts, V);
  id_place_kernel<<<1, 32, 0, s>>>(ids, K, counts, order);
  launch_fill(g, 0.0f, (int64_t)m * V, s);
  id_scatter_dw_kernel<<<(m + 127) / 128, 128, 0, s>>>(e, ids, order, K, m, V, alpha, g);
  return 5;
}

}  // namespace rgb

// ---------------------------------------------------------------------------
// Token tapes (reference data.py:117-207): gather the ids of h'+1 tokens per
// stream (positions planned on the host) into frame-major inputs / targets.
namespace rgb {

__global__ void tape_gather_kernel(const int64_t* corpus, const int64_t* pos, int64_t* inputs, int64_t* targets,
                                   int S, int k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S * (k + 1)) return;
  const int s = i / (k + 1), j = i % (k + 1);
  const int64_t tok = corpus[pos[i]];
  if (j < k) inputs[(int64_t)j * S + s] = tok;
  if (j > 0) targets[(int64_t)(j - 1) * S + s] = tok;
}

void launch_tape_gather(const int64_t* corpus, const int64_t* pos, int64_t* inputs, int64_t* targets, int S, int k,
                        cudaStream_t s) {
  const int n = S * (k + 1);
  if (n > 0) tape_gather_kernel<<<(n + 255) / 256, 256, 0, s>>>(corpus, pos, inputs, targets, S, k);
}

}  // namespace rgb
