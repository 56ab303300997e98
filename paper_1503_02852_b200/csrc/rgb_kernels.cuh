// CUDA kernels of the graph-RNN training step (SIMT fp32 path).
//
//   ew_chain_kernel     elementwise layer ops (activations, gates, f', eps)   K6
//   gemm_nt_kernel      grouped C = sum_seg A_seg * B_seg^T + fused EW chain   K1/K4 (SIMT)
//   gemm_dw_kernel      grouped G = alpha * E^T Y (weight gradients)          K5 (SIMT)
//   softmax_rows_kernel row softmax with mirrored ring write                  K6
//   inject_loss_kernel  delta_out = d - y and per-row loss                    K6
//   sum_rows_kernel     deterministic fp64 loss reduction
//   sgd_kernel          W -= lr * G                                           K6
//   transpose_kernel    W^T refresh (grouped over connections)
#pragma once
#include "rgb_types.cuh"

namespace rgb {

struct TransposeJob {
  float* src;        // [rows x cols] W (updated in place when g is set)
  float* dst;        // [cols x rows] W^T
  const float* g;    // [rows x cols] gradient (null: transpose only)
  int rows, cols;
};
constexpr int kMaxTr = 48;
struct TransposeGroup {
  int njobs;
  float lr;          // W -= lr * g before the transpose (fused SGD)
  int tile_start[kMaxTr + 1];
  int tiles_c[kMaxTr];
  TransposeJob job[kMaxTr];
};

void launch_ew(const EwLaunch& p, cudaStream_t s);
// programmatic dependent launch for the launches that follow (the executor
// enables it inside frame loops); RGB_PDL=0 disables it
void set_pdl_scope(bool on);
bool pdl_active();
// programmatic dependent launch for the launches that follow (the executor
// enables it inside frame loops); RGB_PDL=0 disables it
void set_pdl_scope(bool on);
bool pdl_active();
void launch_gemm_nt(const GemmGroup& p, cudaStream_t s);
void launch_gemm_dw(const DwGroup& p, cudaStream_t s);
// dW of narrow sources (n <= 4, bias edges): two deterministic GEMV passes
// through `part` (dw_narrow_scratch floats); returns the launch count
long long dw_narrow_scratch(const DwGroup& p);
int launch_dw_narrow(const DwGroup& p, float* part, cudaStream_t s);
// tcgen05 (3xTF32, TMEM accumulator) versions of the two GEMM forms; same
// descriptors, tiles recomputed for 128 x {64,128,256} (rgb_tc_gemm.cu).
// returns the number of kernels launched (2 with split-K: GEMM + fixup/epilogue)
int launch_tc_gemm_nt(GemmGroup p, cudaStream_t s);
// split-K scratch (floats) the TMA NT kernel would use for this group (0 = no split)
long long tc_gemm_nt_scratch(const GemmGroup& p);
// tensor-core kernel variants (1 on, 0 off, -1 unchanged): CTA pairs,
// persistent multi-wave kernels, cluster (DSMEM) split-K
void set_tc_config(int pair, int persist, int csplit);
// tensor-core products per k-step: 3 (3xTF32, fp32-exact) or 1 (plain TF32)
void set_tc_terms(int terms);
int get_tc_terms();
void launch_tc_gemm_dw(DwGroup p, cudaStream_t s);
// persistent tensor-core frame loop of a recurrent SCC (rgb_tc_gemm.cu): -1 if
// the loop's GEMM shape does not suit it, else a cudaError_t
int launch_tc_frame_loop(const GemmGroup& g0, const GemmGroup* d_frames, const EwLaunch* d_ew, int n_ew,
                         int fuse_ew, int pattern, const EwLaunch* d_tail, int nframes, unsigned* bar,
                         cudaStream_t s);
void launch_softmax(float* y, int rows, int width, RingWrite ring, bool is_ring, cudaStream_t s);
// target_kind: 0 = int64 class ids, 1 = int32 class ids, 2 = dense fp32 targets.
// criterion: 0 = cross entropy (softmax output), 1 = mse (identity output).
void launch_inject_loss(const float* y, const void* target, int target_kind, int criterion, float* inj,
                        double* row_loss, int rows, int width, int* bad, cudaStream_t s);
void launch_sum_rows(const double* row_loss, int rows, double* out, cudaStream_t s);
// W -= lr * G over n floats and lo = W - trunc_tf32(W); g == nullptr: residual only.
void launch_transpose(const TransposeGroup& p, cudaStream_t s);
void launch_fill(float* p, float v, int64_t n, cudaStream_t s);
void launch_onehot(const int64_t* ids, int rows, int width, float* out, cudaStream_t s);
// token-id input path (rgb_kernels.cu): id history ring, W^T row gather,
// deterministic scatter dW (returns the kernel launch count)
void launch_ids_ring_write(const int64_t* ids, int32_t* ring, int rows, int S, int64_t t_a, int cap, int vocab,
                           int* bad, cudaStream_t s);
void launch_ids_reset(int32_t* ring, int S, int frames, int stream, cudaStream_t s);
void launch_tape_gather(const int64_t* corpus, const int64_t* pos, int64_t* inputs, int64_t* targets, int S, int k,
                        cudaStream_t s);
void launch_gather_rows(const int32_t* ids, const float* wt, float* out, int rows, int n, bool accumulate,
                        cudaStream_t s);
int launch_id_scatter_dw(const float* e, const int32_t* ids, int K, int m, int V, float alpha, float* g, int* scratch,
                         cudaStream_t s);
void launch_count_nonfinite(const float* p, int64_t n, unsigned long long* out, cudaStream_t s);

}  // namespace rgb
