// Per-element layer operations shared by the elementwise kernel and every GEMM
// epilogue (SIMT and tcgen05).  Reference semantics: kernels.py:143-189,
// engine.py:324-349 (forward) and engine.py:519-566 (backward).
#pragma once
#include "rgb_types.cuh"

namespace rgb {

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

__device__ __forceinline__ void ring_store(float* out, int64_t e, int64_t r, int width, bool is_ring,
                                           const RingWrite& ring, float v) {
  out[e] = v;
  if (is_ring) {
    const int64_t moff = ring.frame_rows * width;
    out[e + (r < ring.split ? moff : -moff)] = v;
  }
}

// One elementwise op at (row r, unit j).  `acc` replaces op.base when has_acc.
__device__ __forceinline__ void ew_apply(const EwOp& op, int width, int64_t r, int j, const RingWrite& ring,
                                         bool has_acc, float acc) {
  const int64_t e = r * width + j;
  switch (op.kind) {
    case EW_CONST1:
      ring_store(op.out, e, r, width, op.out_is_ring, ring, 1.0f);
      return;
    case EW_FWD_MUL: {
      float v = op.fac[0][e];
      for (int i = 1; i < op.nfac; ++i) v *= op.fac[i][e];
      ring_store(op.out, e, r, width, op.out_is_ring, ring, v);
      return;
    }
    case EW_FWD_ADD: {
      float v = has_acc ? acc : (op.base ? op.base[e] : 0.0f);
      for (int i = 0; i < op.nterm; ++i) v += op.term[i][e];
      for (int i = 0; i < op.nrank1; ++i) v += op.r1w[i][j] * op.r1src[i][r];
      ring_store(op.out, e, r, width, op.out_is_ring, ring, act_apply(op.act, v));
      return;
    }
    case EW_BWD: {
      float v = has_acc ? acc : (op.base ? op.base[e] : 0.0f);
      for (int i = 0; i < op.nterm; ++i) v += op.term[i][e];
      if (op.act == ACT_SIGMOID || op.act == ACT_TANH) v *= act_deriv(op.act, op.y[e]);
      if (op.inj && r >= op.inj_row0) v += op.inj[(r - op.inj_row0) * width + j];  // after f' (engine.py:548-554)
      op.out[e] = v;
      for (int i = 0; i < op.nfac; ++i) {  // eps_m = delta * prod_{other} z (engine.py:558-566)
        if (!op.eps[i]) continue;
        float p = v;
        for (int k = 0; k < op.nfac; ++k)
          if (k != i) p *= op.fac[k][e];
        op.eps[i][e] = p;
      }
      return;
    }
  }
}

}  // namespace rgb
