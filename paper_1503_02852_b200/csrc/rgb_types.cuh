// Device-side descriptors shared by the executor (rgb_plan.cu) and the kernels.
//
// Every activation / error buffer is row-major [rows x width] fp32 with
// row = frame * S + stream (the reference Batch layout, kernels.py:21-23), so a
// buffer's leading dimension is always its own width and an operand is fully
// described by one pointer to the first row of the step's frame range.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rgb {

enum Act : int { ACT_IDENTITY = 0, ACT_SIGMOID = 1, ACT_TANH = 2, ACT_SOFTMAX = 3 };

// Elementwise layer operations (one per layer and frame range).
enum EwKind : int {
  EW_FWD_ADD = 0,  // y = act(base + sum terms + sum rank1)            (engine.py:334-337)
  EW_FWD_MUL = 1,  // y = prod fac (ascending cid)                      (engine.py:338-348)
  EW_CONST1 = 2,   // y = 1 (non-input layer without anteriors)         (engine.py:331-333)
  EW_BWD = 3,      // delta = (base + sum terms) * f'(y) [+ inj]; eps_m = delta * prod_{other} fac
                   //                                                    (engine.py:519-566)
};

constexpr int kMaxTerms = 4;
constexpr int kMaxRank1 = 3;
constexpr int kMaxFac = 4;
// K depth (fp32) of one TMA stage of the NT tensor-core GEMM: 32 = 128-byte
// rows with SWIZZLE_128B, 16 = 64-byte rows with SWIZZLE_64B.  The tensor
// maps (rgb_plan.cu encode_map) and the UMMA descriptors follow it.
#ifndef RGB_TMA_NT_BK
#define RGB_TMA_NT_BK 32
#endif
constexpr int kTmaNtBk = RGB_TMA_NT_BK;
constexpr int kMaxChain = 6;
constexpr int kMaxSegs = 4;
constexpr int kMaxJobs = 8;
constexpr int kMaxChains = 8;
constexpr int kMaxDw = 48;

struct EwOp {
  int kind, act, nterm, nrank1;
  int nfac, out_is_ring, inj_row0, pad0;
  const float* base;               // nullptr: 0; in a GEMM epilogue the accumulator is the base
  const float* term[kMaxTerms];    // identity-edge operands (same width)
  const float* r1src[kMaxRank1];   // width-1 dense sources: + W[:,0] * src[row]
  const float* r1w[kMaxRank1];
  const float* fac[kMaxFac];       // FWD_MUL factors / BWD co-factors (z of each anterior)
  const float* y;                  // BWD: stored activation for f'
  const float* inj;                // BWD: injected output error, rows >= inj_row0
  float* out;                      // y (forward) or delta (backward)
  float* eps[kMaxFac];             // BWD on a multiplicative layer: eps per anterior
};

// A chain of element-aligned ops over one [rows x width] index space; each
// thread runs the ops in order for its (row, unit), so an op may read what an
// earlier op of the chain wrote at the same (row, unit) without a barrier.
struct EwChain {
  int nops, width;
  EwOp op[kMaxChain];
};

// Ring-buffer mirror bookkeeping of one step: rows < split live in the first
// copy (mirror at +frame_rows*width), rows >= split in the second (mirror at -).
struct RingWrite {
  int64_t split;       // (Cp - slot(t_a)) * S
  int64_t frame_rows;  // Cp * S
};

struct Seg {
  const float* a;      // [rows x K] row-major (K-major A)
  const float* b;      // [N x K] row-major (K-major B): W (forward) or W^T (backward)
  const void* ta;      // TMA tensor map of A's whole buffer (device memory), or null
  const void* tb;      // TMA tensor maps of B and of its tf32 residual B_lo
  const void* tblo;
  int arow;            // row of `a` inside A's buffer (TMA coordinate)
  int k;
};

struct GemmJob {
  int nseg, n;
  Seg seg[kMaxSegs];
  EwChain epi;         // epilogue chain; op 0 takes the accumulator as base
};

struct GemmGroup {
  int njobs, rows;
  int tma, pad;                  // 1: every segment has TMA maps (TMA-fed tcgen05 kernel)
  int tile_start[kMaxJobs + 1];  // prefix sum of tiles per job
  int tiles_n[kMaxJobs];         // tiles along N per job
  RingWrite ring;
  GemmJob job[kMaxJobs];
  // split-K scratch of the TMA tensor-core kernel (owned by the plan): one
  // partial tile per (output tile, split).  part == nullptr: no split.
  float* part;
  long long part_cap;  // floats
  int splits;          // set by launch_tc_gemm_nt
  int pair;            // 1: CTA-pair (cta_group::2) tiles of 256 rows
  int csplit;          // 1: the splits of a tile form a cluster and reduce through DSMEM
  int terms;           // tcgen05 products per k-step: 3 = 3xTF32 (fp32-exact), 1 = plain TF32
};

struct EwLaunch {
  int nchains, rows;
  RingWrite ring;
  EwChain chain[kMaxChains];
};

// dW: G[m, n] = alpha * sum_r E[r, m] * Y[r, n]   (engine.py:578-599, Eq. 19)
struct DwJob {
  const float* e;      // [K x M] (M-major)
  const float* y;      // [K x N] (N-major)
  float* g;            // [M x N] row-major
  int m, n;
  const void* te;      // TMA maps (MN-major boxes) of E's and Y's buffers, or null
  const void* ty;
  int erow, yrow;      // first row of E / Y inside their buffers
};

struct DwGroup {
  int njobs, k;
  float alpha;
  int tma;             // 1: every job has TMA maps
  int terms;           // 3 = 3xTF32 (fp32-exact), 1 = plain TF32
  int tile_start[kMaxDw + 1];
  int tiles_n[kMaxDw];
  DwJob job[kMaxDw];
};

}  // namespace rgb
