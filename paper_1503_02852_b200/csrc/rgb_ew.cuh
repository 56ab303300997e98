// Per-element layer operations shared by the elementwise kernel and every GEMM
// epilogue (SIMT and tcgen05).  Reference semantics: kernels.py:143-189,
// engine.py:324-349 (forward) and engine.py:519-566 (backward).
#pragma once
#include "rgb_types.cuh"

namespace rgb {

// Programmatic dependent launch: kernels of the per-frame loops may be
// launched before their predecessor finishes (prologue overlap); they call
// pdl_wait() before touching global memory the predecessor writes or reads.
// Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// activations (kernels.py:143-189): accurate expf/tanhf, no fast-math

__device__ __forceinline__ float act_apply(int act, float x) {
  if (act == ACT_SIGMOID) return 1.0f / (1.0f + expf(-x));
  if (act == ACT_TANH) return tanhf(x);
  return x;  // identity (softmax is a separate row kernel)
}

// f'(s) from the stored output y (kernels.py:176-189)
__device__ __forceinline__ float act_deriv(int act, float y) {
  if (act == ACT_SIGMOID) return y * (1.0f - y);
  if (act == ACT_TANH) return 1.0f - y * y;
  return 1.0f;  // identity; softmax only ever appears fused with CE (engine.py:537-543)
}

// Operand access policy of ew_apply: DirectMem reads and writes global memory
// only; the recurrent-SCC kernel substitutes a policy that serves operands
// produced earlier in the same loop body from shared memory (rgb_scc.cu).
// Slot ids: terms 0-3, factors 4-7, y 8, base 9; stores: out 0, eps 1-4.
struct DirectMem {
  __device__ __forceinline__ float ld(int, const float* p) const { return *p; }
  __device__ __forceinline__ void st(int, float* p, float v) { *p = v; }
};

template <class M>
__device__ __forceinline__ void ring_store(M& m, float* out, int64_t e, int64_t r, int width, bool is_ring,
                                           const RingWrite& ring, float v) {
  m.st(0, out + e, v);
  if (is_ring) {
    const int64_t moff = ring.frame_rows * width;
    out[e + (r < ring.split ? moff : -moff)] = v;  // mirror copy: never re-read by the writer's chain
  }
}

__device__ __forceinline__ void ring_store(float* out, int64_t e, int64_t r, int width, bool is_ring,
                                           const RingWrite& ring, float v) {
  DirectMem m;
  ring_store(m, out, e, r, width, is_ring, ring, v);
}

// One elementwise op at (row r, unit j).  `acc` replaces op.base when has_acc.
// Every operand load is issued before the first use (predicated, fully
// unrolled over the slot counts): the warp stalls once per op instead of once
// per operand -- the single-stream recurrent loops run these chains on a
// handful of threads, where each stall is a full memory latency.  Summation
// order is unchanged (ascending slots).
//
// KIND / NT / NF >= 0 fix the op kind and the term / factor counts at compile
// time (straight-line code, no per-slot branches: the recurrent-SCC kernel
// dispatches its ops to these, ew_variant below); -1 reads them from the op.
template <int KIND, int NT, int NF, class M>
__device__ __forceinline__ void ew_apply_t(M& m, const EwOp& op, int width, int64_t r, int j, const RingWrite& ring,
                                           bool has_acc, float acc) {
  constexpr int kT = NT >= 0 ? NT : kMaxTerms, kF = NF >= 0 ? NF : kMaxFac;
  constexpr int kR = KIND < 0 ? kMaxRank1 : 0;  // rank-1 terms only on the generic path
  const int64_t e = r * width + j;
  const int kind = KIND >= 0 ? KIND : op.kind;
  const int nterm = NT >= 0 ? NT : op.nterm, nfac = NF >= 0 ? NF : op.nfac;
  if (kind == EW_CONST1) {
    ring_store(m, op.out, e, r, width, op.out_is_ring, ring, 1.0f);
    return;
  }
  const bool mul = kind == EW_FWD_MUL, bwd = kind == EW_BWD;
  float t[kT > 0 ? kT : 1], f[kF > 0 ? kF : 1], rk[kR > 0 ? kR : 1];
#pragma unroll
  for (int i = 0; i < kT; ++i) t[i] = (!mul && i < nterm) ? m.ld(i, op.term[i] + e) : 0.0f;
#pragma unroll
  for (int i = 0; i < kF; ++i) f[i] = ((mul || bwd) && i < nfac) ? m.ld(4 + i, op.fac[i] + e) : 1.0f;
#pragma unroll
  for (int i = 0; i < kR; ++i) rk[i] = (kind == EW_FWD_ADD && i < op.nrank1) ? op.r1w[i][j] * op.r1src[i][r] : 0.0f;
  const float base = (!mul && !has_acc && op.base) ? m.ld(9, op.base + e) : 0.0f;
  const bool fprime = bwd && (op.act == ACT_SIGMOID || op.act == ACT_TANH);
  const float yv = fprime ? m.ld(8, op.y + e) : 0.0f;
  const float inj = (bwd && op.inj && r >= op.inj_row0) ? op.inj[(r - op.inj_row0) * width + j] : 0.0f;
  if (mul) {
    float v = f[0];
#pragma unroll
    for (int i = 1; i < kF; ++i)
      if (i < nfac) v *= f[i];
    ring_store(m, op.out, e, r, width, op.out_is_ring, ring, v);
    return;
  }
  float v = has_acc ? acc : base;
#pragma unroll
  for (int i = 0; i < kT; ++i)
    if (i < nterm) v += t[i];
  if (kind == EW_FWD_ADD) {
#pragma unroll
    for (int i = 0; i < kR; ++i)
      if (i < op.nrank1) v += rk[i];
    ring_store(m, op.out, e, r, width, op.out_is_ring, ring, act_apply(op.act, v));
    return;
  }
  // EW_BWD
  if (fprime) v *= act_deriv(op.act, yv);
  if (op.inj && r >= op.inj_row0) v += inj;  // after f' (engine.py:548-554)
  m.st(0, op.out + e, v);
#pragma unroll
  for (int i = 0; i < kF; ++i) {  // eps_m = delta * prod_{other} z (engine.py:558-566)
    if (i >= nfac || !op.eps[i]) continue;
    float p = v;
#pragma unroll
    for (int k = 0; k < kF; ++k)
      if (k != i && k < nfac) p *= f[k];
    m.st(1 + i, op.eps[i] + e, p);
  }
}

template <class M>
__device__ __forceinline__ void ew_apply(M& m, const EwOp& op, int width, int64_t r, int j, const RingWrite& ring,
                                         bool has_acc, float acc) {
  ew_apply_t<-1, -1, -1>(m, op, width, r, j, ring, has_acc, acc);
}

// Specialised instantiations of ew_apply_t for the op shapes the builders
// emit (LSTM / Elman cells); 0 = generic.
__host__ __device__ __forceinline__ int ew_variant(int kind, int nterm, int nfac, int nrank1) {
  if (kind == EW_CONST1) return 1;
  if (kind == EW_FWD_ADD && nrank1 == 0 && nterm <= 2) return 2 + nterm;         // 2..4
  if (kind == EW_FWD_MUL && (nfac == 2 || nfac == 3)) return 3 + nfac;            // 5, 6
  if (kind == EW_BWD && nterm <= 2 && (nfac == 0 || nfac == 2)) return 7 + nterm + (nfac ? 3 : 0);  // 7..12
  return 0;
}

template <class M>
__device__ __forceinline__ void ew_apply_variant(int var, M& m, const EwOp& op, int width, int64_t r, int j,
                                                 const RingWrite& ring, bool has_acc, float acc) {
  switch (var) {
    case 1: ew_apply_t<EW_CONST1, 0, 0>(m, op, width, r, j, ring, has_acc, acc); break;
    case 2: ew_apply_t<EW_FWD_ADD, 0, 0>(m, op, width, r, j, ring, has_acc, acc); break;
    case 3: ew_apply_t<EW_FWD_ADD, 1, 0>(m, op, width, r, j, ring, has_acc, acc); break;
    case 4: ew_apply_t<EW_FWD_ADD, 2, 0>(m, op, width, r, j, ring, has_acc, acc); break;
    case 5: ew_apply_t<EW_FWD_MUL, 0, 2>(m, op, width, r, j, ring, has_acc, acc); break;
    case 6: ew_apply_t<EW_FWD_MUL, 0, 3>(m, op, width, r, j, ring, has_acc, acc); break;
    case 7: ew_apply_t<EW_BWD, 0, 0>(m, op, width, r, j, ring, has_acc, acc); break;
    case 8: ew_apply_t<EW_BWD, 1, 0>(m, op, width, r, j, ring, has_acc, acc); break;
    case 9: ew_apply_t<EW_BWD, 2, 0>(m, op, width, r, j, ring, has_acc, acc); break;
    case 10: ew_apply_t<EW_BWD, 0, 2>(m, op, width, r, j, ring, has_acc, acc); break;
    case 11: ew_apply_t<EW_BWD, 1, 2>(m, op, width, r, j, ring, has_acc, acc); break;
    case 12: ew_apply_t<EW_BWD, 2, 2>(m, op, width, r, j, ring, has_acc, acc); break;
    default: ew_apply_t<-1, -1, -1>(m, op, width, r, j, ring, has_acc, acc); break;
  }
}

__device__ __forceinline__ void ew_apply(const EwOp& op, int width, int64_t r, int j, const RingWrite& ring,
                                         bool has_acc, float acc) {
  DirectMem m;
  ew_apply(m, op, width, r, j, ring, has_acc, acc);
}

// The same op over U independent elements at once.  Every operand stream is
// gathered for all U elements before anything is stored, so one op costs one
// memory latency per operand instead of one per element -- the GEMM epilogues
// run on a single CTA per SM and cannot hide latency with more warps.
template <int U>
__device__ __forceinline__ void ew_apply_batch(const EwOp& op, int width, const int64_t (&r)[U], const int (&j)[U],
                                               const bool (&ok)[U], const RingWrite& ring, bool has_acc,
                                               const float (&acc)[U]) {
  int64_t e[U];
  float v[U], t[U];
#pragma unroll
  for (int u = 0; u < U; ++u) e[u] = r[u] * width + j[u];
  const int kind = op.kind;
  if (kind == EW_CONST1) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) ring_store(op.out, e[u], r[u], width, op.out_is_ring, ring, 1.0f);
    return;
  }
  if (kind == EW_FWD_MUL) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ok[u] ? op.fac[0][e[u]] : 0.0f;
    for (int i = 1; i < op.nfac; ++i) {
#pragma unroll
      for (int u = 0; u < U; ++u) t[u] = ok[u] ? op.fac[i][e[u]] : 0.0f;
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] *= t[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) ring_store(op.out, e[u], r[u], width, op.out_is_ring, ring, v[u]);
    return;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = has_acc ? acc[u] : ((op.base && ok[u]) ? op.base[e[u]] : 0.0f);
  for (int i = 0; i < op.nterm; ++i) {
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = ok[u] ? op.term[i][e[u]] : 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] += t[u];
  }
  if (kind == EW_FWD_ADD) {
    for (int i = 0; i < op.nrank1; ++i) {
#pragma unroll
      for (int u = 0; u < U; ++u) t[u] = ok[u] ? op.r1w[i][j[u]] * op.r1src[i][r[u]] : 0.0f;
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] += t[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) ring_store(op.out, e[u], r[u], width, op.out_is_ring, ring, act_apply(op.act, v[u]));
    return;
  }
  // EW_BWD
  if (op.act == ACT_SIGMOID || op.act == ACT_TANH) {
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = ok[u] ? op.y[e[u]] : 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] *= act_deriv(op.act, t[u]);
  }
  if (op.inj) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      t[u] = (ok[u] && r[u] >= op.inj_row0) ? op.inj[(r[u] - op.inj_row0) * width + j[u]] : 0.0f;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] += t[u];
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (ok[u]) op.out[e[u]] = v[u];
  if (op.nfac == 0) return;
  // eps_m = delta * prod_{other} z: gather every factor once, then form the products
  float f[kMaxFac][U];  // fully unrolled: stays in registers
#pragma unroll
  for (int i = 0; i < kMaxFac; ++i) {
#pragma unroll
    for (int u = 0; u < U; ++u) f[i][u] = (i < op.nfac && ok[u]) ? op.fac[i][e[u]] : 1.0f;
  }
#pragma unroll
  for (int i = 0; i < kMaxFac; ++i) {
    if (i >= op.nfac || !op.eps[i]) continue;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float p = v[u];
#pragma unroll
      for (int k = 0; k < kMaxFac; ++k)
        if (k != i) p *= f[k][u];
      if (ok[u]) op.eps[i][e[u]] = p;
    }
  }
}

// ---------------------------------------------------------------------------
// Row-vectorised form for the tensor-core epilogues: R rows x 4 consecutive
// units (j % 4 == 0) per thread, every operand moved as one 16-byte access.
// Valid when width % 4 == 0 and every pointer of the chain is 16-B aligned
// (chain_vec_ok); per element the arithmetic is exactly ew_apply's.

__device__ __forceinline__ float4 ld4(const float* p, int64_t e) { return *reinterpret_cast<const float4*>(p + e); }
__device__ __forceinline__ void st4(float* p, int64_t e, float4 v) { *reinterpret_cast<float4*>(p + e) = v; }
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 mul4(float4 a, float4 b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }

__device__ __forceinline__ void ring_store4(float* out, int64_t e, int64_t r, int width, bool is_ring,
                                            const RingWrite& ring, float4 v) {
  st4(out, e, v);
  if (is_ring) {
    const int64_t moff = ring.frame_rows * width;
    st4(out, e + (r < ring.split ? moff : -moff), v);
  }
}

__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// true when the whole chain can take the 16-byte path
__device__ __forceinline__ bool chain_vec_ok(const EwChain& ch, int width) {
  if (width % 4) return false;
  for (int k = 0; k < ch.nops; ++k) {
    const EwOp& o = ch.op[k];
    bool ok = aligned16(o.out) && aligned16(o.base) && aligned16(o.y) && aligned16(o.inj);
    for (int i = 0; i < kMaxTerms; ++i) ok = ok && aligned16(o.term[i]);
    for (int i = 0; i < kMaxRank1; ++i) ok = ok && aligned16(o.r1w[i]);
    for (int i = 0; i < kMaxFac; ++i) ok = ok && aligned16(o.fac[i]) && aligned16(o.eps[i]);
    if (!ok) return false;
  }
  return true;
}

template <int R>
__device__ __forceinline__ void ew_apply_vec(const EwOp& op, int width, const int64_t (&r)[R], int j,
                                             const bool (&ok)[R], const RingWrite& ring, bool has_acc,
                                             const float4 (&acc)[R]) {
  int64_t e[R];
  float4 v[R], t[R];
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int u = 0; u < R; ++u) e[u] = r[u] * width + j;
  const int kind = op.kind;
  if (kind == EW_CONST1) {
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, make_float4(1.f, 1.f, 1.f, 1.f));
    return;
  }
  if (kind == EW_FWD_MUL) {
    float4 ff[kMaxFac][R];
#pragma unroll
    for (int i = 0; i < kMaxFac; ++i) {
#pragma unroll
      for (int u = 0; u < R; ++u) ff[i][u] = (i < op.nfac && ok[u]) ? ld4(op.fac[i], e[u]) : zero;
    }
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = ff[0][u];
#pragma unroll
    for (int i = 1; i < kMaxFac; ++i) {
      if (i >= op.nfac) break;
#pragma unroll
      for (int u = 0; u < R; ++u) v[u] = mul4(v[u], ff[i][u]);
    }
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, v[u]);
    return;
  }
  // all term loads first (one stall per op, not per operand); ascending sum
  float4 tt[kMaxTerms][R];
#pragma unroll
  for (int i = 0; i < kMaxTerms; ++i) {
#pragma unroll
    for (int u = 0; u < R; ++u) tt[i][u] = (i < op.nterm && ok[u]) ? ld4(op.term[i], e[u]) : zero;
  }
#pragma unroll
  for (int u = 0; u < R; ++u) v[u] = has_acc ? acc[u] : ((op.base && ok[u]) ? ld4(op.base, e[u]) : zero);
#pragma unroll
  for (int i = 0; i < kMaxTerms; ++i) {
    if (i >= op.nterm) break;
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = add4(v[u], tt[i][u]);
  }
  if (kind == EW_FWD_ADD) {
    for (int i = 0; i < op.nrank1; ++i) {
      const float4 w = ld4(op.r1w[i], j);
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const float s = ok[u] ? op.r1src[i][r[u]] : 0.0f;
        v[u] = add4(v[u], make_float4(w.x * s, w.y * s, w.z * s, w.w * s));
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const float4 a = make_float4(act_apply(op.act, v[u].x), act_apply(op.act, v[u].y),
                                   act_apply(op.act, v[u].z), act_apply(op.act, v[u].w));
      if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, a);
    }
    return;
  }
  // EW_BWD
  if (op.act == ACT_SIGMOID || op.act == ACT_TANH) {
#pragma unroll
    for (int u = 0; u < R; ++u) t[u] = ok[u] ? ld4(op.y, e[u]) : zero;
#pragma unroll
    for (int u = 0; u < R; ++u)
      v[u] = mul4(v[u], make_float4(act_deriv(op.act, t[u].x), act_deriv(op.act, t[u].y),
                                    act_deriv(op.act, t[u].z), act_deriv(op.act, t[u].w)));
  }
  if (op.inj) {
#pragma unroll
    for (int u = 0; u < R; ++u)
      t[u] = (ok[u] && r[u] >= op.inj_row0) ? ld4(op.inj, (r[u] - op.inj_row0) * width + j) : zero;
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = add4(v[u], t[u]);
  }
#pragma unroll
  for (int u = 0; u < R; ++u)
    if (ok[u]) st4(op.out, e[u], v[u]);
  if (op.nfac == 0) return;
  float4 f[kMaxFac][R];
  const float4 one = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
  for (int i = 0; i < kMaxFac; ++i) {
#pragma unroll
    for (int u = 0; u < R; ++u) f[i][u] = (i < op.nfac && ok[u]) ? ld4(op.fac[i], e[u]) : one;
  }
#pragma unroll
  for (int i = 0; i < kMaxFac; ++i) {
    if (i >= op.nfac || !op.eps[i]) continue;
#pragma unroll
    for (int u = 0; u < R; ++u) {
      float4 p = v[u];
#pragma unroll
      for (int k = 0; k < kMaxFac; ++k)
        if (k != i) p = mul4(p, f[k][u]);
      if (ok[u]) st4(op.eps[i], e[u], p);
    }
  }
}

// Specialised vector op (KIND, NT terms, NF factors fixed at compile time,
// ew_variant ids 2-12): every operand of the op -- terms, base, y, injection
// and the co-factors -- is loaded before its first store (the co-factors
// belong to other layers, never to this op's out / eps), so the op costs one
// memory latency; with the counts known the register arrays hold only what
// the op uses.  Arithmetic per element is exactly ew_apply's.
template <int R, int KIND, int NT, int NF>
__device__ __forceinline__ void ew_apply_vec_t(const EwOp& op, int width, const int64_t (&r)[R], int j,
                                               const bool (&ok)[R], const RingWrite& ring, bool has_acc,
                                               const float4 (&acc)[R]) {
  int64_t e[R];
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f), one = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
  for (int u = 0; u < R; ++u) e[u] = r[u] * width + j;
  if constexpr (KIND == EW_CONST1) {
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, one);
    return;
  } else {
    constexpr bool kBwd = KIND == EW_BWD, kMul = KIND == EW_FWD_MUL;
    // bx: the base (FWD_ADD without accumulator) or the stored y for f' (BWD);
    // BWD ops with a base or an injection take the generic path (dispatcher)
    float4 tt[NT > 0 ? NT : 1][R], ff[NF > 0 ? NF : 1][R], bx[R];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
#pragma unroll
      for (int u = 0; u < R; ++u) tt[i][u] = ok[u] ? ld4(op.term[i], e[u]) : zero;
    }
#pragma unroll
    for (int i = 0; i < NF; ++i) {
#pragma unroll
      for (int u = 0; u < R; ++u) ff[i][u] = ok[u] ? ld4(op.fac[i], e[u]) : one;
    }
    const bool has_base = KIND == EW_FWD_ADD && !has_acc && op.base;
    const bool fprime = kBwd && (op.act == ACT_SIGMOID || op.act == ACT_TANH);
#pragma unroll
    for (int u = 0; u < R; ++u)
      bx[u] = (has_base && ok[u]) ? ld4(op.base, e[u]) : ((fprime && ok[u]) ? ld4(op.y, e[u]) : zero);
    float4 v[R];
    if constexpr (kMul) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        v[u] = ff[0][u];
#pragma unroll
        for (int i = 1; i < NF; ++i) v[u] = mul4(v[u], ff[i][u]);
        if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, v[u]);
      }
      return;
    } else {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        v[u] = has_acc ? acc[u] : (kBwd ? zero : bx[u]);
#pragma unroll
        for (int i = 0; i < NT; ++i) v[u] = add4(v[u], tt[i][u]);
      }
      if constexpr (KIND == EW_FWD_ADD) {
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const float4 a = make_float4(act_apply(op.act, v[u].x), act_apply(op.act, v[u].y),
                                       act_apply(op.act, v[u].z), act_apply(op.act, v[u].w));
          if (ok[u]) ring_store4(op.out, e[u], r[u], width, op.out_is_ring, ring, a);
        }
        return;
      } else {
#pragma unroll
        for (int u = 0; u < R; ++u) {
          if (fprime)
            v[u] = mul4(v[u], make_float4(act_deriv(op.act, bx[u].x), act_deriv(op.act, bx[u].y),
                                          act_deriv(op.act, bx[u].z), act_deriv(op.act, bx[u].w)));
          if (ok[u]) st4(op.out, e[u], v[u]);
        }
#pragma unroll
        for (int i = 0; i < NF; ++i) {  // eps_m = delta * prod_{other} z (engine.py:558-566)
          if (!op.eps[i]) continue;
#pragma unroll
          for (int u = 0; u < R; ++u) {
            float4 p = v[u];
#pragma unroll
            for (int k = 0; k < NF; ++k)
              if (k != i) p = mul4(p, ff[k][u]);
            if (ok[u]) st4(op.eps[i], e[u], p);
          }
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void ew_apply_vec_variant(const EwOp& op, int width, const int64_t (&r)[R], int j,
                                                     const bool (&ok)[R], const RingWrite& ring, bool has_acc,
                                                     const float4 (&acc)[R]) {
  int var = ew_variant(op.kind, op.nterm, op.nfac, op.nrank1);
  if (op.kind == EW_BWD && (op.inj || (op.base && !has_acc))) var = 0;
  switch (var) {
    case 1: ew_apply_vec_t<R, EW_CONST1, 0, 0>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 2: ew_apply_vec_t<R, EW_FWD_ADD, 0, 0>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 3: ew_apply_vec_t<R, EW_FWD_ADD, 1, 0>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 4: ew_apply_vec_t<R, EW_FWD_ADD, 2, 0>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 5: ew_apply_vec_t<R, EW_FWD_MUL, 0, 2>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 6: ew_apply_vec_t<R, EW_FWD_MUL, 0, 3>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 7: ew_apply_vec_t<R, EW_BWD, 0, 0>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 8: ew_apply_vec_t<R, EW_BWD, 1, 0>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 9: ew_apply_vec_t<R, EW_BWD, 2, 0>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 10: ew_apply_vec_t<R, EW_BWD, 0, 2>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 11: ew_apply_vec_t<R, EW_BWD, 1, 2>(op, width, r, j, ok, ring, has_acc, acc); break;
    case 12: ew_apply_vec_t<R, EW_BWD, 2, 2>(op, width, r, j, ok, ring, has_acc, acc); break;
    default:
      if constexpr (R > 4 && R % 4 == 0) {
        // generic ops in quarters of 4 rows: the generic form's operand arrays at
        // R = 8 would spill
#pragma unroll 1
        for (int h = 0; h < R; h += 4) {
          int64_t rh[4];
          bool okh[4];
          float4 acch[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) rh[u] = r[h + u], okh[u] = ok[h + u], acch[u] = acc[h + u];
          ew_apply_vec<4>(op, width, rh, j, okh, ring, has_acc, acch);
        }
      } else {
        ew_apply_vec<R>(op, width, r, j, ok, ring, has_acc, acc);
      }
      break;
  }
}

// the whole chain on R rows x 4 units; op 0 takes `acc` (GEMM epilogues).
// Latency note: every op waits for its own operand loads, so the callers
// give each thread as many rows (R) as registers allow -- one memory latency
// per op covers all of them.
template <int R, bool SPEC = true>
__device__ __forceinline__ void ew_chain_vec(const EwChain& ch, int width, const int64_t (&r)[R], int j,
                                             const bool (&ok)[R], const RingWrite& ring, bool has_acc,
                                             const float4 (&acc)[R]) {
  // SPEC: specialised single-latency ops (latency-bound per-frame epilogues);
  // the persistent GEMM's epilogue overlaps other tiles and keeps the lean
  // generic form (no spills at its 136-register budget)
  for (int k = 0; k < ch.nops; ++k) {
    if constexpr (SPEC)
      ew_apply_vec_variant<R>(ch.op[k], width, r, j, ok, ring, has_acc && k == 0, acc);
    else
      ew_apply_vec<R>(ch.op[k], width, r, j, ok, ring, has_acc && k == 0, acc);
  }
}

}  // namespace rgb
