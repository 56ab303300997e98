// Persistent recurrent-SCC kernel (paper §3.1: the frame-sequential part).
//
// One launch runs a whole per-frame loop of one strongly connected component
// -- forward (ascending) or backward (descending) -- instead of one or two
// launches per frame.  The loop body is the same int32 step program the host
// executor interprets (schedule.py):
//   * at kernel start the body is parsed ONCE into shared-memory templates
//     (GEMM jobs, elementwise chains) plus a list of frame-dependent pointer
//     "slots" (operand buffer + frame shift); per frame the CTA's threads
//     re-resolve the slots in parallel -- no per-frame parsing;
//   * GEMM step (the intra-SCC dense edges, e.g. cell(t-1) -> {in,forget}
//     gates): CTA b owns output columns [b*W/G, (b+1)*W/G) of every job; the
//     matching rows of the recurrent weights (W_rec) are loaded into shared
//     memory once and stay resident for all frames.  Phase 1: one warp per
//     (job, stream row) reads the A row once and dots it with every owned
//     weight row; phase 2: one thread per output element runs the fused
//     elementwise chain (activation, gates, cell update, f', eps);
//   * elementwise step: the CTA's own columns (element-local by construction);
//   * before every GEMM step the CTAs synchronise: the hardware cluster
//     barrier (~0.2 us, measured) when the SCC is small enough for one cluster
//     of <= 16 CTAs, else an atomic grid barrier (~2.3 us) over a cooperative
//     launch (tools/barrier_probe.cu).
// Reference semantics: engine.py:405-413 (forward), 568-576 (backward).
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>

#include "rgb_ew.cuh"
#include "rgb_kernels.cuh"
#include "rgb_scc.cuh"

namespace rgb {

#ifdef RGB_EXP_TRACE
// tuning aid: clock64 marks of CTA 0 / thread 0 for the first frames (tools/trace_scc.py)
__device__ long long g_scc_trace[64][16];
__device__ long long g_scc_pro[8];
#define SCC_MARK(f, k) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && (f) < 64) g_scc_trace[f][k] = clock64();
#define SCC_PRO(k) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_scc_pro[k] = clock64();
#else
#define SCC_MARK(f, k)
#define SCC_PRO(k)
#endif

namespace {

constexpr int kColChunk = 4;   // owned weight rows dotted per pass over an A row
constexpr int kMaxSteps = 8;
constexpr int kMaxSlots = 512;
enum { S_EW = 1, S_GEMM = 2 };

__device__ __forceinline__ long long pmod_d(long long a, long long m) { return ((a % m) + m) % m; }

struct SJob {
  int nseg, n;
  const float* a[kMaxSegs];   // A rows of the frame (slot-resolved)
  const float* bs[kMaxSegs];  // this CTA's weight rows (shared or global)
  const float* bsrc[kMaxSegs];  // the same rows in global memory (cache source)
  int k[kMaxSegs];
  int ldb[kMaxSegs];  // row stride of bs: round4(K) + 4 in the cache (conflict-free float4 rows), K in global
  int boff[kMaxSegs];  // offset of bs in the shared weight cache (floats)
  short cid[kMaxSegs], trans[kMaxSegs];
};

__host__ __device__ __forceinline__ int round4(int k) { return (k + 3) & ~3; }

struct Slot {
  int off;      // byte offset of the pointer field inside the template arena
  short buf, shift;
  short inj;    // 1: only valid on injected frames (t > t0)
  short kind;   // SL_READ (element-indexed operand), SL_WRITE, SL_ROW (rank-1 source); SL_EXT: read of
                // a buffer the loop body never writes (prefetchable)
};
enum { SL_READ = 0, SL_WRITE = 1, SL_ROW = 2, SL_EXT = 3 };
constexpr int kMaxBufBits = 2048;

// Forwarded chain values.  Every op carries 16 code bytes: [0..9] the source
// of each operand slot (terms 0-3, factors 4-7, y 8, base 9), [10..14]
// the value index its stores (out, eps 0-3) also write, [15] its ew_variant.  kMem = global
// memory; otherwise a row of the CTA's shared `vals` array, optionally
// (kPrev) holding the previous frame's value.
constexpr unsigned char kMem = 0xFF, kPrev = 0x40;
constexpr int kMaxRecs = 64;
constexpr int kMaxExt = 32;
constexpr int kTcacheMagic = 0x5cc7e301;
struct ExtRow {  // an operand the body reads but never writes: staged per frame into vals row `row`
  short buf, shift, row;
};
struct ChainCode {
  unsigned char c[kMaxChain][16];
};
struct OpRec {  // build-time record of one op of the body (thread 0 only)
  short step, chain, k;
  short rb[10], rs[10];  // read slots: buffer (-1 none), frame shift
  short wb[5];           // written buffers (out, eps 0-3), -1 none
  unsigned char* code;
};

// ew_apply policy: operands produced earlier in the body by this CTA come from
// shared memory instead of a global-memory round trip.  The value for local
// element `el` lives in vals[idx * stride + el]; every (buffer, frame) is
// written by exactly one op, so a row holds exactly what memory holds.
struct SccVals {
  const unsigned char* code;
  float* vals;
  int el, stride;
  bool first;  // first frame of the launch: previous-frame rows are not filled yet
  __device__ __forceinline__ float ld(int s, const float* p) const {
    const unsigned cd = code[s];
    if (cd != kMem && !(first && (cd & kPrev))) return vals[(cd & 0x3F) * stride + el];
    return *p;
  }
  __device__ __forceinline__ void st(int s, float* p, float v) {
    *p = v;
    const unsigned cd = code[10 + s];
    if (cd != kMem) vals[cd * stride + el] = v;
  }
};

struct Step {
  int kind, n;          // S_GEMM: n jobs; S_EW: n chains
  int jobs_off, chains_off, codes_off;
  int slot_begin, slot_end;
  int pf_end;           // prefetch range [slot_begin, pf_end): up to the next CTA barrier
};

// Per-frame index bases: ring slot, window index, chunk index of frame t.
struct FrameIdx {
  int tmod, win, chunk, inj;
};

__device__ __forceinline__ float* resolve(const SccCtx& c, const SccBuf* bufs, const FrameIdx& f, int buf, int shift) {
  const SccBuf b = bufs[buf];
  int idx;
  if (b.kind == 0) {
    idx = f.tmod + shift;
    while (idx < 0) idx += c.cap;
    while (idx >= c.cap) idx -= c.cap;
  } else {
    idx = (b.kind == 1 ? f.win : f.chunk) + shift;
  }
  return c.ws + b.off + (long long)idx * c.S * b.width;
}

// ---- one-time template build (thread 0) ------------------------------------

struct Builder {
  const int32_t* w;
  int pos;
  unsigned char* arena;
  int used;
  Slot* slots;
  int nslots;
  bool ok;
  OpRec* recs;
  int nrec, step, nchain;
  short* writer;  // per buffer: rec * 5 + store slot of its only writer, -1 none, -2 several
  bool has_r1;    // an op holds frame-independent rank-1 weight pointers (no template caching)
  __device__ void wrote(int b, int x) {
    if (b < 0 || b >= kMaxBufBits || nrec > kMaxRecs) return;
    writer[b] = writer[b] == -1 ? (short)((nrec - 1) * 5 + x) : (short)-2;
  }

  template <class T>
  __device__ T* alloc(int count, int& off) {
    used = (used + 15) & ~15;
    off = used;
    used += count * (int)sizeof(T);
    return reinterpret_cast<T*>(arena + off);
  }
  __device__ void slot(const void* field, int buf, int shift, int inj = 0, int kind = SL_READ) {
    if (nslots >= kMaxSlots) {
      ok = false;
      return;
    }
    slots[nslots++] = Slot{(int)(reinterpret_cast<const unsigned char*>(field) - arena), (short)buf, (short)shift,
                           (short)inj, (short)kind};
  }
  __device__ void op(const SccCtx& c, const SccBuf* bufs, const SccW* wts, EwOp& o, int k, unsigned char* code) {
    OpRec dummy;  // past kMaxRecs ops: nrec > kMaxRecs disables forwarding
    OpRec& R = nrec < kMaxRecs ? recs[nrec] : dummy;
    ++nrec;
    R.step = (short)step;
    R.chain = (short)nchain;
    R.k = (short)k;
    R.code = code;
    for (int i = 0; i < 10; ++i) R.rb[i] = -1, R.rs[i] = 0;
    for (int i = 0; i < 5; ++i) R.wb[i] = -1;
    for (int i = 0; i < 16; ++i) code[i] = kMem;
    o.kind = w[pos++];
    o.act = w[pos++];
    const int out = w[pos++];
    o.out = nullptr;
    slot(&o.out, out, 0, 0, SL_WRITE);
    R.wb[0] = (short)out;
    wrote(out, 0);
    o.out_is_ring = bufs[out].kind == 0;
    o.nterm = w[pos++];
    for (int i = 0; i < o.nterm; ++i, pos += 2) {
      slot(&o.term[i], w[pos], w[pos + 1]);
      R.rb[i] = (short)w[pos], R.rs[i] = (short)w[pos + 1];
    }
    o.nrank1 = w[pos++];
    if (o.nrank1 > 0) has_r1 = true;
    for (int i = 0; i < o.nrank1; ++i, pos += 3) {
      slot(&o.r1src[i], w[pos], w[pos + 1], 0, SL_ROW);
      o.r1w[i] = c.w + wts[w[pos + 2]].off;  // frame-independent
    }
    o.nfac = w[pos++];
    for (int i = 0; i < o.nfac; ++i, pos += 2) {
      slot(&o.fac[i], w[pos], w[pos + 1]);
      R.rb[4 + i] = (short)w[pos], R.rs[4 + i] = (short)w[pos + 1];
    }
    o.y = nullptr;
    if (w[pos] >= 0) {
      slot(&o.y, w[pos], w[pos + 1]);
      R.rb[8] = (short)w[pos], R.rs[8] = (short)w[pos + 1];
    }
    pos += 2;
    o.base = nullptr;  // -2 (accumulator) stays null
    if (w[pos] >= 0) {
      slot(&o.base, w[pos], w[pos + 1]);
      R.rb[9] = (short)w[pos], R.rs[9] = (short)w[pos + 1];
    }
    pos += 2;
    o.inj = nullptr;
    o.inj_row0 = 0;
    if (w[pos++]) slot(&o.inj, c.inj_buf, 0, 1);
    const int neps = w[pos++];
    for (int i = 0; i < kMaxFac; ++i) o.eps[i] = nullptr;
    code[15] = (unsigned char)ew_variant(o.kind, o.nterm, o.nfac, o.nrank1);
    for (int i = 0; i < neps; ++i, ++pos)
      if (w[pos] >= 0) {
        slot(&o.eps[i], w[pos], 0, 0, SL_WRITE);
        R.wb[1 + i] = (short)w[pos];
        wrote(w[pos], 1 + i);
      }
  }
  __device__ void chain(const SccCtx& c, const SccBuf* bufs, const SccW* wts, EwChain& ch, ChainCode& cc) {
    ch.width = w[pos++];
    ch.nops = w[pos++];
    for (int k = 0; k < ch.nops; ++k) op(c, bufs, wts, ch.op[k], k, cc.c[k]);
    ++nchain;
  }
};

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

__device__ __forceinline__ void sync_ctas(const SccCtx& c, unsigned& my_gen) {
  if (c.cluster) {
    // release/acquire at cluster scope: global writes of every CTA in the
    // cluster are visible after the barrier (the acquire invalidates L1)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    grid_barrier(c.bar, c.bar + 1, gridDim.x, my_gen);
  }
}

// Rows [rg, rg + nr) (nr <= RB) of one output column `col` of job J over the
// ks-th of KS slices of every K segment: float4 shared-memory reads (A rows
// broadcast across the warp, padded B rows conflict-free), RB accumulators in
// registers; partial sums go to outp[r * QT].
template <int RB>
__device__ __forceinline__ void dots_rows(const SJob& J, const float* wcache, const float* ablk, int nrow, int rg,
                                          int nr, int col, int ks, int KS, float* outp, int QT) {
  float acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = 0.0f;
  for (int s = 0; s < J.nseg; ++s) {
    const int K4 = round4(J.k[s]) / 4;
    const int kb = (int)((long long)ks * K4 / KS), ke = (int)((long long)(ks + 1) * K4 / KS);
    const float4* b4 = reinterpret_cast<const float4*>(wcache + J.boff[s] + col * J.ldb[s]);
    const float4* a4 = reinterpret_cast<const float4*>(ablk + rg * K4 * 4);
    ablk += nrow * K4 * 4;
#pragma unroll 4
    for (int k = kb; k < ke; ++k) {
      const float4 bv = b4[k];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (RB == 1 || r < nr) {
          const float4 av = a4[r * K4 + k];
          acc[r] = fmaf(av.x, bv.x, acc[r]);
          acc[r] = fmaf(av.y, bv.y, acc[r]);
          acc[r] = fmaf(av.z, bv.z, acc[r]);
          acc[r] = fmaf(av.w, bv.w, acc[r]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r)
    if (r < nr) outp[(long long)r * QT] = acc[r];
}

__global__ void __launch_bounds__(kSccThreads, 1) scc_kernel(const __grid_constant__ SccCtx c) {
  extern __shared__ __align__(16) unsigned char sm[];
  // layout: [tables][weight cache][accumulators][A stage][forwarded values][template arena][slots]
  SccBuf* sbufs = reinterpret_cast<SccBuf*>(sm);
  SccW* swts = reinterpret_cast<SccW*>(sbufs + c.nbufs);
  float* wcache = reinterpret_cast<float*>(
      sm + ((sizeof(SccBuf) * c.nbufs + sizeof(SccW) * c.nwts + 15) & ~size_t(15)));
  float* accs = wcache + ((c.wcache_floats + 3) & ~3LL);
  float* astage = accs + ((c.acc_floats + 3) & ~3LL);
  float* vals = astage + ((c.stage_floats + 3) & ~3LL);
  unsigned char* arena = reinterpret_cast<unsigned char*>(vals + ((c.vals_floats + 3) & ~3LL));
  Slot* slots = reinterpret_cast<Slot*>(arena + c.arena_bytes);
  __shared__ Step steps[kMaxSteps];
  __shared__ int s_nsteps;
  __shared__ unsigned s_wbits[kMaxBufBits / 32];
  __shared__ OpRec s_recs[kMaxRecs];
  __shared__ short s_pend[kMaxRecs * 10];
  __shared__ short s_writer[kMaxBufBits];
  __shared__ int s_nrec, s_next;
  __shared__ ExtRow s_ext[kMaxExt];
  __shared__ int s_cached, s_nslots, s_cacheable;

  SCC_PRO(0)
  for (int i = threadIdx.x; i < c.nbufs; i += blockDim.x) sbufs[i] = c.bufs[i];
  for (int i = threadIdx.x; i < kMaxBufBits; i += blockDim.x) s_writer[i] = -1;
  for (int i = threadIdx.x; i < c.nwts; i += blockDim.x) swts[i] = c.wts[i];
  // CTA (rb, cb): streams [r0, r1) x units [j0, j1).  Streams never exchange
  // data, so only the ncb CTAs of one row block synchronise (one cluster each).
  const int W = c.width;
  const int cb = blockIdx.x % c.ncb, rb = blockIdx.x / c.ncb;
  const int j0 = (int)((long long)cb * W / c.ncb);
  const int j1 = (int)((long long)(cb + 1) * W / c.ncb);
  const int ncol = j1 - j0;
  const int r0 = (int)((long long)rb * c.S / c.nrb), r1 = (int)((long long)(rb + 1) * c.S / c.nrb);
  const int nrow = r1 - r0;
  __syncthreads();

  // ---- template image: [header 16 B][arena][slots][steps][read-only rows]
  const long long img_arena = 16, img_slots = img_arena + ((c.arena_bytes + 15) & ~15LL);
  const long long img_steps = img_slots + ((sizeof(Slot) * kMaxSlots + 15) & ~size_t(15));
  const long long img_ext = img_steps + ((sizeof(Step) * kMaxSteps + 15) & ~size_t(15));
  if (threadIdx.x == 0) s_cached = c.tcache && *reinterpret_cast<volatile int*>(c.tcache) == kTcacheMagic;
  __syncthreads();
  if (s_cached) {
    // a previous launch of this body built the templates: copy them in
    const int* hdr = reinterpret_cast<const int*>(c.tcache);
    for (long long i = threadIdx.x; i < c.arena_bytes / 4; i += blockDim.x)
      reinterpret_cast<int*>(arena)[i] = reinterpret_cast<const int*>(c.tcache + img_arena)[i];
    for (int i = threadIdx.x; i < hdr[3] * (int)(sizeof(Slot) / 4); i += blockDim.x)
      reinterpret_cast<int*>(slots)[i] = reinterpret_cast<const int*>(c.tcache + img_slots)[i];
    for (int i = threadIdx.x; i < (int)(sizeof(Step) * kMaxSteps / 4); i += blockDim.x)
      reinterpret_cast<int*>(steps)[i] = reinterpret_cast<const int*>(c.tcache + img_steps)[i];
    for (int i = threadIdx.x; i < kMaxExt; i += blockDim.x)
      s_ext[i] = reinterpret_cast<const ExtRow*>(c.tcache + img_ext)[i];
    if (threadIdx.x == 0) {
      s_nsteps = hdr[1];
      s_next = hdr[2];
    }
    __syncthreads();
    // per-CTA / per-launch fields: this CTA's weight rows and their place in
    // the shared cache (ncol differs between CTAs when ncb does not divide W)
    if (threadIdx.x == 0) {
      int woff = 0;
      for (int si = 0; si < s_nsteps; ++si) {
        if (steps[si].kind != S_GEMM) continue;
        SJob* jobs = reinterpret_cast<SJob*>(arena + steps[si].jobs_off);
        for (int jb = 0; jb < steps[si].n; ++jb)
          for (int s = 0; s < jobs[jb].nseg; ++s) {
            SJob& J = jobs[jb];
            J.bsrc[s] = (J.trans[s] ? c.wt : c.w) + swts[J.cid[s]].off + (long long)j0 * J.k[s];
            if (c.use_cache) {
              J.boff[s] = woff;
              J.bs[s] = wcache + woff;
              woff += ncol * J.ldb[s];
            } else {
              J.bs[s] = J.bsrc[s];
            }
          }
      }
    }
  } else {
  // ---- build the templates once (thread 0), preload W_rec rows (all threads)
  if (threadIdx.x == 0) {
    Builder B{c.body, 0, arena, 0, slots, 0, true, s_recs, 0, 0, 0, s_writer, false};
    int nsteps = 0, woff = 0;
    while (B.pos < c.body_len && nsteps < kMaxSteps) {
      Step& st = steps[nsteps++];
      st.kind = B.w[B.pos++];
      st.n = B.w[B.pos++];
      st.slot_begin = B.nslots;
      B.step = nsteps - 1;
      if (st.kind == S_GEMM) {
        SJob* jobs = B.alloc<SJob>(st.n, st.jobs_off);
        EwChain* chains = B.alloc<EwChain>(st.n, st.chains_off);
        ChainCode* codes = B.alloc<ChainCode>(st.n, st.codes_off);
        for (int jb = 0; jb < st.n; ++jb) {
          SJob& J = jobs[jb];
          J.nseg = B.w[B.pos++];
          for (int s = 0; s < J.nseg; ++s, B.pos += 4) {
            const int ab = B.w[B.pos], ash = B.w[B.pos + 1], cid = B.w[B.pos + 2], trans = B.w[B.pos + 3];
            const SccW wd = swts[cid];
            const int K = trans ? wd.rows : wd.cols;
            J.k[s] = K;
            J.a[s] = nullptr;
            B.slot(&J.a[s], ab, ash);
            J.bsrc[s] = (trans ? c.wt : c.w) + wd.off + (long long)j0 * K;
            J.cid[s] = (short)cid;
            J.trans[s] = (short)trans;
            if (c.use_cache) {
              J.bs[s] = wcache + woff;
              J.boff[s] = woff;
              J.ldb[s] = round4(K) + 4;
              woff += ncol * J.ldb[s];
            } else {
              J.bs[s] = J.bsrc[s];
              J.ldb[s] = K;
            }
          }
          B.chain(c, sbufs, swts, chains[jb], codes[jb]);
          J.n = chains[jb].width;
        }
      } else {
        st.jobs_off = 0;
        EwChain* chains = B.alloc<EwChain>(st.n, st.chains_off);
        ChainCode* codes = B.alloc<ChainCode>(st.n, st.codes_off);
        for (int i = 0; i < st.n; ++i) B.chain(c, sbufs, swts, chains[i], codes[i]);
      }
      st.slot_end = B.nslots;
    }
    s_nsteps = nsteps;
    // reads of buffers the body never writes can be prefetched into L1 right
    // after a CTA barrier (the barrier's acquire is what would drop them)
    unsigned* wbits = s_wbits;
    for (int i = 0; i < kMaxBufBits / 32; ++i) wbits[i] = 0;
    for (int i = 0; i < B.nslots; ++i)
      if (slots[i].kind == SL_WRITE && slots[i].buf < kMaxBufBits) wbits[slots[i].buf >> 5] |= 1u << (slots[i].buf & 31);
    for (int i = 0; i < B.nslots; ++i)
      if (slots[i].kind == SL_READ && slots[i].buf < kMaxBufBits && !(wbits[slots[i].buf >> 5] >> (slots[i].buf & 31) & 1))
        slots[i].kind = SL_EXT;
    for (int si = 0; si < nsteps; ++si) {
      int e = si + 1;
      while (e < nsteps && steps[e].kind != S_GEMM) ++e;
      steps[si].pf_end = e < nsteps ? steps[e].slot_begin : B.nslots;
    }
    s_nrec = B.nrec;
    s_next = 0;
    s_nslots = B.nslots;
    s_cacheable = B.ok && !B.has_r1;
  }
  __syncthreads();
  SCC_PRO(1)
  // forwarding: a read of (buffer, frame) written by exactly one op of the
  // body is served from `vals` when that write is already done when the read
  // runs -- same frame: an earlier step, or an earlier op of the same chain
  // (same thread); previous frame: a later step, or a later-or-same op of the
  // same chain (not yet overwritten this frame).  Ops of different chains in
  // one step run concurrently on other threads: memory.  Pass 1 (all
  // threads) finds the writer of every read slot, pass 2 (thread 0, body
  // order) numbers the value rows.
  if (s_nrec <= kMaxRecs) {
    const int prev = c.reverse ? 1 : -1;
    const int nrec = s_nrec;
    for (int q = threadIdx.x; q < nrec * 10; q += blockDim.x) {
      const OpRec& R = s_recs[q / 10];
      const int sl = q % 10;
      short found = -1;
      const int b = R.rb[sl];
      if (b >= 0 && b < kMaxBufBits && s_writer[b] >= 0 && (R.rs[sl] == 0 || R.rs[sl] == prev)) {
        const int wr = s_writer[b] / 5, wsl = s_writer[b] % 5;
        {
          const OpRec& Wr = s_recs[wr];
          const bool ok = R.rs[sl] == 0 ? (Wr.step < R.step || (Wr.chain == R.chain && Wr.k < R.k))
                                        : (Wr.step > R.step || (Wr.chain == R.chain && Wr.k >= R.k));
          if (ok) found = (short)(wr * 5 + wsl);
        }
      }
      s_pend[q] = found;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int nv = 0, next = 0;
      for (int r = 0; r < nrec; ++r) {
        OpRec& R = s_recs[r];
        for (int sl = 0; sl < 10; ++sl) {
          const int b = R.rb[sl];
          if (b < 0) continue;
          const int sh = R.rs[sl], pend = s_pend[r * 10 + sl];
          if (pend < 0) {
            // never written by the body: staged into a row at every frame start
            if (b >= kMaxBufBits || (s_wbits[b >> 5] >> (b & 31) & 1)) continue;
            int row = -1;
            for (int x = 0; x < next; ++x)
              if (s_ext[x].buf == b && s_ext[x].shift == sh) row = s_ext[x].row;
            if (row < 0) {
              if (nv >= c.vals_cap || next >= kMaxExt) continue;
              row = nv++;
              s_ext[next++] = ExtRow{(short)b, (short)sh, (short)row};
            }
            R.code[sl] = (unsigned char)row;
            continue;
          }
          unsigned char& dst = s_recs[pend / 5].code[10 + pend % 5];
          if (dst == kMem) {
            if (nv >= c.vals_cap) continue;
            dst = (unsigned char)nv++;
          }
          R.code[sl] = (unsigned char)(dst | (sh == 0 ? 0 : kPrev));
        }
      }
      s_next = next;
    }
  }
  __syncthreads();
  if (c.tcache && blockIdx.x == 0 && s_cacheable) {
    // publish the templates for the next launches of this body
    for (long long i = threadIdx.x; i < c.arena_bytes / 4; i += blockDim.x)
      reinterpret_cast<int*>(c.tcache + img_arena)[i] = reinterpret_cast<const int*>(arena)[i];
    for (int i = threadIdx.x; i < s_nslots * (int)(sizeof(Slot) / 4); i += blockDim.x)
      reinterpret_cast<int*>(c.tcache + img_slots)[i] = reinterpret_cast<const int*>(slots)[i];
    for (int i = threadIdx.x; i < (int)(sizeof(Step) * kMaxSteps / 4); i += blockDim.x)
      reinterpret_cast<int*>(c.tcache + img_steps)[i] = reinterpret_cast<const int*>(steps)[i];
    for (int i = threadIdx.x; i < kMaxExt; i += blockDim.x)
      reinterpret_cast<ExtRow*>(c.tcache + img_ext)[i] = s_ext[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      int* hdr = reinterpret_cast<int*>(c.tcache);
      hdr[1] = s_nsteps;
      hdr[2] = s_next;
      hdr[3] = s_nslots;
      __threadfence();
      atomicExch(hdr, kTcacheMagic);
    }
  }
  }  // built here
  __syncthreads();
  SCC_PRO(2)
  // everything above reads only the plan's own tables: with programmatic
  // dependent launch it overlaps the tail of the preceding kernel
  pdl_wait();
  if (c.use_cache) {
    int off = 0;
    for (int si = 0; si < s_nsteps; ++si) {
      if (steps[si].kind != S_GEMM) continue;
      const SJob* jobs = reinterpret_cast<const SJob*>(arena + steps[si].jobs_off);
      for (int jb = 0; jb < steps[si].n; ++jb)
        for (int s = 0; s < jobs[jb].nseg; ++s) {
          const int K = jobs[jb].k[s], ld = jobs[jb].ldb[s];
          const float* src = jobs[jb].bsrc[s];
          if ((K & 3) == 0 && (reinterpret_cast<size_t>(src) & 15) == 0) {
            // float4 rows, 8 loads in flight per thread before the stores
            const int k4 = K / 4, l4 = ld / 4, n4 = ncol * k4;
            for (int i0 = threadIdx.x; i0 < n4; i0 += 8 * blockDim.x) {
              float4 v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (i0 + u * (int)blockDim.x < n4) v[u] = reinterpret_cast<const float4*>(src)[i0 + u * blockDim.x];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < n4) reinterpret_cast<float4*>(wcache + off)[(i / k4) * l4 + i % k4] = v[u];
              }
            }
            for (int i = threadIdx.x; i < ncol; i += blockDim.x)  // zero row pads
              reinterpret_cast<float4*>(wcache + off)[i * l4 + k4] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            for (int i = threadIdx.x; i < ncol * ld; i += blockDim.x) {
              const int cc = i / ld, kk = i - cc * ld;
              wcache[off + i] = kk < K ? src[(long long)cc * K + kk] : 0.0f;
            }
          }
          off += ncol * ld;
        }
    }
  }
  unsigned my_gen = 0;
  if (!c.cluster && threadIdx.x == 0) my_gen = *reinterpret_cast<volatile unsigned*>(c.bar + 1);
  __syncthreads();

  SCC_PRO(3)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int f = 0; f < c.frames; ++f) {
    const long long t = c.reverse ? c.t_first + c.frames - 1 - f : c.t_first + f;
    FrameIdx fi;
    fi.tmod = (int)pmod_d(t, c.cap);
    fi.win = (int)(t - c.t1 + c.hmax - 1);
    fi.chunk = (int)(t - c.chunk_base);
    fi.inj = t > c.t0;
    RingWrite ring;
    ring.split = (long long)(c.cap - fi.tmod) * c.S;
    ring.frame_rows = (long long)c.cap * c.S;
    SCC_MARK(f, 0)
    // stage this frame's read-only operands into their vals rows, overlapped
    // with the first CTA barrier (split arrive / wait on a cluster)
    const bool g0 = steps[0].kind == S_GEMM;
    if (g0 && c.cluster) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    {
      const int nel = nrow * ncol;
      const int nq = s_next * nel;
      if (nq <= (int)blockDim.x) {  // one element per thread (single stream rows)
        const int q = threadIdx.x;
        if (q < nq) {
          const int x = q / nel, el = q - x * nel;
          const ExtRow er = s_ext[x];
          const int srow = r0 + el / ncol, col = el - (el / ncol) * ncol;
          const float* base = resolve(c, sbufs, fi, er.buf, er.shift);
          vals[er.row * c.vals_stride + el] = base[(long long)srow * sbufs[er.buf].width + j0 + col];
        }
      } else
      for (int q0 = threadIdx.x; q0 < nq; q0 += 8 * blockDim.x) {
        float v[8];  // all loads in flight before the stores
        int dst[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = q0 + u * blockDim.x;
          dst[u] = -1;
          if (q < nq) {
            const int x = q / nel, el = q - x * nel;
            const ExtRow er = s_ext[x];
            const int srow = r0 + el / ncol, col = el - (el / ncol) * ncol;
            const float* base = resolve(c, sbufs, fi, er.buf, er.shift);
            v[u] = base[(long long)srow * sbufs[er.buf].width + j0 + col];
            dst[u] = er.row * c.vals_stride + el;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (dst[u] >= 0) vals[dst[u]] = v[u];
      }
    }
    if (g0) {
      if (c.cluster)
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      else
        grid_barrier(c.bar, c.bar + 1, gridDim.x, my_gen);
    }
    for (int si = 0; si < s_nsteps; ++si) {
      const Step st = steps[si];
      // the CTAs only exchange data through the dense (GEMM) reads
      SCC_MARK(f, 1 + si * 5)
      if (st.kind == S_GEMM && si > 0) sync_ctas(c, my_gen);
      SCC_MARK(f, 2 + si * 5)
      if (si == 0 || st.kind == S_GEMM) {
        // resolve the frame's pointers up to the next barrier
        for (int i = st.slot_begin + threadIdx.x; i < st.pf_end; i += blockDim.x) {
          const Slot sl = slots[i];
          *reinterpret_cast<float**>(arena + sl.off) =
              (sl.inj && !fi.inj) ? nullptr : resolve(c, sbufs, fi, sl.buf, sl.shift);
        }
        __syncthreads();
      }
      const EwChain* chains = reinterpret_cast<const EwChain*>(arena + st.chains_off);
      const ChainCode* codes = reinterpret_cast<const ChainCode*>(arena + st.codes_off);
      SccVals m{nullptr, vals, 0, c.vals_stride, f == 0};
      if (st.kind == S_GEMM) {
        const SJob* jobs = reinterpret_cast<const SJob*>(arena + st.jobs_off);
        // stage the A rows of this row block once (rows padded to round4(K),
        // zero tail): every CTA reads the state its peers wrote last phase
        const float* a_src[kMaxJobs][kMaxSegs];
        int lda[kMaxJobs][kMaxSegs];
        // (one stream row: the warp-per-column-chunk loop below is faster)
        const bool fast = c.stage_floats > 0 && c.use_cache && nrow >= 2;
        if (c.stage_floats > 0) {
          int off = 0;
          for (int jb = 0; jb < st.n; ++jb)
            for (int s = 0; s < jobs[jb].nseg; ++s) {
              const int K = jobs[jb].k[s], ld = round4(K);
              const float* src = jobs[jb].a[s] + (long long)r0 * K;
              if ((K & 3) == 0 && ((reinterpret_cast<size_t>(src) & 15) == 0)) {
                const int n4 = nrow * K / 4;
                for (int i0 = threadIdx.x; i0 < n4; i0 += 4 * blockDim.x) {
                  float4 v[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    if (i0 + u * (int)blockDim.x < n4) v[u] = reinterpret_cast<const float4*>(src)[i0 + u * blockDim.x];
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    if (i0 + u * (int)blockDim.x < n4) reinterpret_cast<float4*>(astage + off)[i0 + u * blockDim.x] = v[u];
                }
              } else {
                for (int i = threadIdx.x; i < nrow * ld; i += blockDim.x) {
                  const int r = i / ld, k = i - r * ld;
                  astage[off + i] = k < K ? src[(long long)r * K + k] : 0.0f;
                }
              }
              a_src[jb][s] = astage + off;
              lda[jb][s] = ld;
              off += nrow * ld;
            }
          __syncthreads();
        } else {
          for (int jb = 0; jb < st.n; ++jb)
            for (int s = 0; s < jobs[jb].nseg; ++s) {
              a_src[jb][s] = jobs[jb].a[s] + (long long)r0 * jobs[jb].k[s];
              lda[jb][s] = jobs[jb].k[s];
            }
        }
        SCC_MARK(f, 3 + si * 5)
        // accs: [row][q], q = job * ncol + unit (QT columns in all)
        const int QT = st.n * ncol;
        if (fast) {
          // register-blocked SIMT dots: thread (q, ks) owns output column q
          // for up to 8 rows over the ks-th K slice of every segment; float4
          // smem reads (A broadcast across the warp, padded B rows
          // conflict-free); the KS partials are summed through smem
          int NQ = 1;
          while (NQ < QT && NQ < 128) NQ <<= 1;  // kSccThreads = 3 * 128
          const int KS = blockDim.x / NQ;
          const int tq = threadIdx.x % NQ, ks = threadIdx.x / NQ;
          for (int q = tq; q < QT; q += NQ) {
            const int jb = q / ncol, col = q - jb * ncol;
            const SJob& J = jobs[jb];
            int aoff0 = 0;  // this job's first A block in astage (offsets, not pointers:
            for (int x = 0; x < jb; ++x)  // keeps the loads in the shared window, LDS.128)
              for (int s = 0; s < jobs[x].nseg; ++s) aoff0 += nrow * round4(jobs[x].k[s]);
            for (int rg = 0; rg < nrow; rg += 12) {
              const int nr = min(12, nrow - rg);
              float* outp = accs + ((long long)ks * nrow + rg) * QT + q;
              if (nr == 1)
                dots_rows<1>(J, wcache, astage + aoff0, nrow, rg, 1, col, ks, KS, outp, QT);
              else if (nr == 2)
                dots_rows<2>(J, wcache, astage + aoff0, nrow, rg, 2, col, ks, KS, outp, QT);
              else if (nr <= 4)
                dots_rows<4>(J, wcache, astage + aoff0, nrow, rg, nr, col, ks, KS, outp, QT);
              else if (nr <= 8)
                dots_rows<8>(J, wcache, astage + aoff0, nrow, rg, nr, col, ks, KS, outp, QT);
              else
                dots_rows<12>(J, wcache, astage + aoff0, nrow, rg, nr, col, ks, KS, outp, QT);
            }
          }
          __syncthreads();
          if (KS > 1) {
            for (int o = threadIdx.x; o < nrow * QT; o += blockDim.x) {
              float v = accs[o];
              for (int x = 1; x < KS; ++x) v += accs[(long long)x * nrow * QT + o];
              accs[o] = v;
            }
            __syncthreads();
          }
        } else {
          // generic: one warp per (job, row, chunk of owned columns), lanes over K
          const int nchunks = (ncol + kColChunk - 1) / kColChunk;
          const int items1 = st.n * nrow * nchunks;
          for (int it = warp; it < items1; it += nwarps) {
            const int jb = it / (nrow * nchunks), rem = it - jb * (nrow * nchunks);
            const int r = rem / nchunks, c0 = (rem - r * nchunks) * kColChunk;
            const SJob& J = jobs[jb];
            float part[kColChunk];
#pragma unroll
            for (int q = 0; q < kColChunk; ++q) part[q] = 0.f;
            for (int s = 0; s < J.nseg; ++s) {
              const float* a = a_src[jb][s] + (long long)r * lda[jb][s];
              const float* b = J.bs[s] + (long long)c0 * J.ldb[s];
              const int K = J.k[s], ldb = J.ldb[s];
#pragma unroll 4
              for (int k = lane; k < K; k += 32) {
                const float av = a[k];
#pragma unroll
                for (int q = 0; q < kColChunk; ++q)
                  if (c0 + q < ncol) part[q] = fmaf(av, b[(long long)q * ldb + k], part[q]);
              }
            }
#pragma unroll
            for (int q = 0; q < kColChunk; ++q) {
#pragma unroll
              for (int o = 16; o; o >>= 1) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
            }
            if (lane == 0) {
#pragma unroll
              for (int q = 0; q < kColChunk; ++q)
                if (c0 + q < ncol) accs[(long long)r * QT + jb * ncol + c0 + q] = part[q];
            }
          }
          __syncthreads();
        }
        SCC_MARK(f, 4 + si * 5)
        const int items = nrow * QT;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
          const int r = it / QT, q = it - r * QT;
          const int jb = q / ncol, col = q - jb * ncol;
          const EwChain& ch = chains[jb];
          const float acc = accs[it];
          m.el = r * ncol + col;
          for (int k = 0; k < ch.nops; ++k) {
            m.code = codes[jb].c[k];
            ew_apply_variant(m.code[15], m, ch.op[k], ch.width, r0 + r, j0 + col, ring, k == 0, acc);
            SCC_MARK(f, 6 + k + si * 5)
          }
        }
      } else {
        const int items = nrow * ncol;
        for (int i = 0; i < st.n; ++i) {
          const EwChain& ch = chains[i];
          for (int e = threadIdx.x; e < items; e += blockDim.x) {
            const int srow = r0 + e / ncol, col = j0 + (e - (e / ncol) * ncol);
            m.el = e;
            for (int k = 0; k < ch.nops; ++k) {
              m.code = codes[i].c[k];
              ew_apply_variant(m.code[15], m, ch.op[k], ch.width, srow, col, ring, false, 0.0f);
            }
          }
        }
      }
      __syncthreads();
      SCC_MARK(f, 5 + si * 5)
    }
  }
  if (c.cluster) {  // no CTA may exit while a peer could still be inside a barrier phase
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

}  // namespace

size_t scc_smem_bytes(const SccCtx& c) {
  return ((sizeof(SccBuf) * c.nbufs + sizeof(SccW) * c.nwts + 15) & ~size_t(15)) +
         (size_t)((c.wcache_floats + 3) & ~3LL) * 4 + (size_t)((c.acc_floats + 3) & ~3LL) * 4 +
         (size_t)((c.stage_floats + 3) & ~3LL) * 4 + (size_t)((c.vals_floats + 3) & ~3LL) * 4 + c.arena_bytes + sizeof(Slot) * kMaxSlots + 64;
}

bool scc_tcache_fits(long long arena_bytes) {
  return 16 + ((arena_bytes + 15) & ~15LL) + (long long)((sizeof(Slot) * kMaxSlots + 15) & ~size_t(15)) +
             (long long)((sizeof(Step) * kMaxSteps + 15) & ~size_t(15)) + (long long)sizeof(ExtRow) * kMaxExt <=
         kSccTcacheBytes;
}

size_t scc_arena_bytes(int max_jobs_total, int max_chains_total) {
  const size_t b = (size_t)max_jobs_total * (sizeof(SJob) + 16) +
                   (size_t)max_chains_total * (sizeof(EwChain) + sizeof(ChainCode) + 32) + 64;
  return (b + 15) & ~size_t(15);  // the slot table follows the arena
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

static int g_scc_pdl = [] {
  const char* e = getenv("RGB_SCC_PDL");
  return e ? atoi(e) : 1;
}();

int scc_max_clusters(int ncb, size_t smem) {
  cudaFuncSetAttribute(scc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(scc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncb);
  cfg.blockDim = dim3(kSccThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ncb;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, scc_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return n < 1 ? 1 : n;
}

cudaError_t launch_scc(const SccCtx& c, int blocks, size_t smem, cudaStream_t s) {
  // the attribute is per function, not per launch: (re)set it for this size
  cudaError_t e = cudaFuncSetAttribute(scc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (c.cluster) {
    e = cudaFuncSetAttribute(scc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(c.threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c.ncb;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = g_scc_pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, scc_kernel, c);
  }
  void* args[] = {const_cast<SccCtx*>(&c)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(scc_kernel), dim3(blocks), dim3(c.threads), args,
                                     smem, s);
}

}  // namespace rgb

#ifdef RGB_EXP_TRACE
extern "C" int rgb_exp_scc_trace(long long* out) {
  if (cudaMemcpyFromSymbol(out + 64 * 16, rgb::g_scc_pro, sizeof(rgb::g_scc_pro)) != cudaSuccess) return 3;
  return cudaMemcpyFromSymbol(out, rgb::g_scc_trace, sizeof(rgb::g_scc_trace)) == cudaSuccess ? 0 : 3;
}
#endif
