/* rnngraph_b200.h -- C ABI of the B200-native graph-RNN BPTT(h; h') training step.
 *
 * Drop-in boundary for the forward / backward / update path of the reference
 * package `rnngraph` (arXiv 1503.02852).  The reference has no FFI: its
 * boundary is the Python API in /root/reference/pkg/src/rnngraph/engine.py.
 * Each entry point below replaces one of those functions; the Python mirror
 * (paper_1503_02852_b200/engine.py) binds them with ctypes exactly as a
 * maintainer would.
 *
 * Conventions
 *  - All tensors are caller-owned fp32 device buffers (plain pointers); the
 *    plan owns only its parsed schedule.  The activation history, error
 *    buffers and scratch live in ONE caller-allocated device workspace whose
 *    size rgb_plan_workspace_bytes() reports and whose internal layout is
 *    fixed by the schedule program (emitted by paper_1503_02852_b200/schedule.py).
 *  - Weights: one flat fp32 buffer W of n_params floats: every dense
 *    connection's (dst_size x src_size) row-major matrix at the offset the
 *    program's weight table gives; a same-layout buffer WT holding the
 *    transposes (the reference keeps the same cache, engine.py:111-139); and
 *    a gradient buffer G of n_params floats.  (The 3xTF32 tensor-core GEMMs
 *    form the tf32 residuals of their operands in shared memory.)
 *  - Work is enqueued on `stream` (a cudaStream_t); nothing synchronises
 *    except rgb_read_loss().
 *  - Every function returns RGB_OK (0) or an error code; rgb_last_error()
 *    returns the thread-local message of the last failure.  No CPU fallback:
 *    rgb_plan_create() fails when no sm_100 device is present.
 */
#ifndef RNNGRAPH_B200_H
#define RNNGRAPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGB_ABI_VERSION 1

enum rgb_status {
  RGB_OK = 0,
  RGB_ERR_ENGINE = 1,  /* guard violation -> EngineError (engine.py:86-87) */
  RGB_ERR_KERNEL = 2,  /* shape / argument misuse -> KernelError (kernels.py:54-55) */
  RGB_ERR_CUDA = 3,    /* CUDA runtime failure or no sm_100 device */
  RGB_ERR_FLOAT = 4    /* non-finite values -> FloatingPointError (kernels.py:344-348) */
};

typedef struct rgb_plan rgb_plan;

int rgb_abi_version(void);
const char* rgb_last_error(void);

/* Parse a schedule program (int32 words emitted by schedule.py) for one
 * network, stream count S and BPTT horizon h.  Replaces the per-call
 * schedule walk of forward_chunk/backward_window (engine.py:405-413,
 * 568-576) and StreamState's layout (engine.py:197-229). */
int rgb_plan_create(const int32_t* program, int64_t n_words, rgb_plan** out);
int rgb_plan_destroy(rgb_plan* plan);
int rgb_plan_workspace_bytes(const rgb_plan* plan, int64_t* bytes);
/* Bind a zero-filled device workspace of at least workspace_bytes. */
int rgb_plan_bind(rgb_plan* plan, void* workspace);
int rgb_plan_get_cursor(const rgb_plan* plan, int64_t* cursor);
int rgb_plan_set_cursor(rgb_plan* plan, int64_t cursor);

/* forward_chunk (engine.py:352-418): advance every stream by `frames`
 * frames.  `x` is (frames*S, n_in) fp32, frame-major; x_on_host != 0 means
 * a host pointer (copied inside this call).  sequential != 0 runs the
 * paper's frame-by-frame baseline schedule (frame_parallel=False). */
int rgb_forward_chunk(rgb_plan* plan, const float* w, const float* x, int x_on_host, int frames,
                      int sequential, void* stream);

/* forward_chunk with token-id inputs (engine.py:308-316, 372-403): `ids` is
 * (frames*S) int64, frame-major, in [0, n_in) (host pointer if ids_on_host).
 * The plan keeps an id history instead of one-hot rows: dense edges out of
 * the input layer gather rows of W^T (hence `wt`), and backward_window
 * computes their gradient as a deterministic sorted scatter (kernels.py:
 * 106-140).  A plan is in id mode from its first id chunk on. */
int rgb_forward_chunk_ids(rgb_plan* plan, const float* w, const float* wt, const int64_t* ids, int ids_on_host,
                          int frames, int sequential, void* stream);

/* inject_output_error + loss_value (engine.py:425-474) for the newest
 * `frames` frames: delta_out = d - y into the plan's injection buffer and
 * the summed loss into the plan's device loss slot.  target_kind: 0 int64
 * class ids, 1 int32 class ids, 2 dense fp32 (frames*S, n_out).
 * criterion: 0 cross-entropy/softmax, 1 mse/identity. */
int rgb_inject_output_error(rgb_plan* plan, const void* target, int target_kind, int target_on_host,
                            int criterion, int frames, void* stream);
/* Read the last loss (synchronises the stream).  Fails with RGB_ERR_ENGINE
 * when an input id or a target class id of an earlier step was out of range
 * (the kernels substitute a zero row / a NaN loss and raise a sticky flag;
 * the reference raises EngineError / IndexError, engine.py:385-389, 443-456). */
int rgb_read_loss(rgb_plan* plan, double* loss, void* stream);
/* The same out-of-range check without reading the loss (synchronises). */
int rgb_check_inputs(rgb_plan* plan, void* stream);
/* Enqueue the copy of the last loss into `dst` (pinned host or device memory)
 * without synchronising; the caller waits on the stream / an event. */
int rgb_read_loss_async(rgb_plan* plan, double* dst, void* stream);
/* Copy the plan's injection buffer rows in/out (frames*S, n_out), device
 * pointers; used when the caller supplies its own delta_out. */
int rgb_set_injection(rgb_plan* plan, const float* delta_out, int frames, void* stream);
int rgb_get_injection(rgb_plan* plan, float* delta_out, int frames, void* stream);

/* Plan-free inject_output_error / loss_value on arbitrary (rows, width)
 * output rows: delta = d - y, per-row loss into row_loss[rows] (fp64
 * scratch) and their fixed-order sum into *loss (device). */
int rgb_inject_rows(const float* y, const void* target, int target_kind, int criterion, float* delta,
                    double* row_loss, double* loss, int rows, int width, void* stream);

/* Device-fed token tapes (reference data.py:117-207): gather the ids at
 * corpus positions pos[(n_streams, h_prime + 1)] (planned by the host tape
 * cursors) into frame-major inputs and one-ahead targets, (h_prime*n_streams)
 * int64 each. */
int rgb_tape_gather(const int64_t* corpus, const int64_t* pos, int64_t* inputs, int64_t* targets, int n_streams,
                    int h_prime, void* stream);

/* Token-id chunk -> dense one-hot rows (rows, width) on the device; id -1
 * gives a zero row.  Feeds forward_chunk's id-input mode (engine.py:372-403;
 * bitwise equal to one-hot dense input in the reference, test_engine.py:277-312). */
int rgb_onehot_rows(const int64_t* ids, int rows, int width, float* out, void* stream);

/* backward_window (engine.py:481-599) for the window (t1-h, t1], t1 = the
 * cursor, errors injected on (t1-h', t1].  Writes the loss gradient
 * dE/dW (= -sum eps y^T, engine.py:13-21) into G for every dense edge. */
int rgb_backward_window(rgb_plan* plan, const float* wt, float* g, int h, int h_prime, int sequential,
                        void* stream);

/* ---- Multi-GPU: stream-sharded data parallelism -------
 * One process per GPU, each owning a slice of the S streams; the only exchange
 * is the SUM of the weight gradients over the GPUs (the reference folds the
 * per-stream partials in one process, engine.py:593-598).  NCCL is loaded at
 * run time (dlopen of libnccl.so.2, the copy PyTorch maps; RGB_NCCL_LIB
 * overrides).  Rank 0 draws the 128-byte unique id, the caller ships it to
 * the other ranks (e.g. through the torch.distributed store). */
typedef struct rgb_comm rgb_comm;
int rgb_comm_unique_id(void* id_out /* 128 bytes */);
int rgb_comm_init(const void* id /* 128 bytes */, int nranks, int rank, rgb_comm** out);
int rgb_comm_destroy(rgb_comm* comm);
int rgb_comm_size(const rgb_comm* comm, int* nranks, int* rank);
/* In-place SUM of n fp32 gradients over all ranks (one flat buffer). */
int rgb_allreduce_grads(rgb_comm* comm, float* g, int64_t n, void* stream);
/* In-place SUM (op_max = 0) or MAX (op_max = 1) of n doubles (loss, timings). */
int rgb_allreduce_f64(rgb_comm* comm, double* v, int64_t n, int op_max, void* stream);
/* backward_window with the gradient exchange overlapped: the dW of the edges
 * into each supernode is computed right after that supernode's backward
 * (reverse topological order) and summed over the ranks on a communication
 * stream while the supernodes below are backpropagated; the call's stream
 * waits for every bucket before returning control of G.  comm == NULL runs
 * the same bucketed schedule without communication. */
int rgb_backward_window_allreduce(rgb_plan* plan, const float* wt, float* g, int h, int h_prime, rgb_comm* comm,
                                  void* stream);

/* sgd_update (engine.py:606-612): W -= lr*G fused with the WT = W^T refresh. */
int rgb_sgd_update(rgb_plan* plan, float* w, float* wt, const float* g, float lr, void* stream);
/* Weights.refresh (engine.py:138-139): WT = W^T. */
int rgb_refresh_transpose(rgb_plan* plan, const float* w, float* wt, void* stream);

/* StreamState.reset_stream (engine.py:267-276). */
int rgb_reset_stream(rgb_plan* plan, int stream_index, void* stream);

/* Read-only view of one schedule buffer over frames [t_lo, t_hi] (frame-major
 * rows of `width` floats, contiguous): activation rings (layer y, edge z) at
 * the current cursor, or the error buffers of the backward window that ended
 * at the current cursor (the last rgb_backward_window or its replay) -- the
 * per-layer deltas and the per-edge eps of multiplicative destinations that
 * the reference computes as locals of backward_window (engine.py:512-566).
 * Buffer ids come from the program's buffer table (schedule.Layout). */
int rgb_window_view(const rgb_plan* plan, int buffer, int64_t t_lo, int64_t t_hi, const float** ptr, int* width);

/* Count non-finite values of one buffer over frames [t_lo, t_hi] (the
 * check_finite guard, engine.py:415-417); result copied to *count (sync). */
int rgb_count_nonfinite(rgb_plan* plan, int buffer, int64_t t_lo, int64_t t_hi, int64_t* count, void* stream);

/* GEMM engine: 0 auto (tcgen05 3xTF32 above a work threshold, SIMT fp32
 * for latency-bound small products), 1 SIMT only, 2 tcgen05 only.  The
 * reference's deterministic k-ascending GEMMs are kernels.py:84-103. */
int rgb_set_gemm_mode(int mode);
/* Persistent recurrent-SCC kernel: 1 (default) runs every eligible
 * frame-sequential loop (engine.py:405-413, 568-576) as one cooperative launch
 * with W_rec resident in shared memory and a grid barrier per dense
 * dependency; 0 launches the loop body once per frame. */
int rgb_set_scc_mode(int on);
/* Persistent tensor-core frame loops: 1 (default) runs every recurrent loop
 * whose body is one tensor-core sized GEMM step plus elementwise steps (the
 * large-S LSTM / stacked-LSTM SCCs, engine.py:405-413, 568-576) as one
 * cooperative launch over all its frames with a grid barrier per dependent
 * step; 0 launches the body once per frame
 * (with programmatic dependent launch; DESIGN.md §9 compares the two). */
int rgb_set_frame_loop(int on);
/* Cross-layer wavefront: the stages between persistent SCC
 * loops of a forward / backward section run on their own streams over frame
 * blocks (default on; env RGB_WAVEFRONT=0 or rgb_set_wavefront(0) disables).
 * No reference counterpart (schedule switch; results equal within fp32). */
int rgb_set_wavefront(int on);
/* Stand-alone GEMM forms (kernel-level parity tests): C[m,n] = A[m,k] . B[n,k]
 * (both row-major) and G[m,n] = alpha * sum_r E[r,m] Y[r,n]; mode 1 SIMT,
 * 2 tcgen05. */
int rgb_gemm_nt(const float* a, const float* b, float* c, int m, int n, int k, int mode, void* stream);
int rgb_gemm_dw(const float* e, const float* y, float* g, int m, int n, int k, float alpha, int mode, void* stream);
/* mode 3 of rgb_gemm_dw: the TMA-fed tcgen05 kernels (m, n multiples of 32). */
/* TMA-fed tcgen05 form of rgb_gemm_nt; b_lo = b - trunc_tf32(b) (k % 4 == 0). */
int rgb_gemm_nt_tma(const float* a, const float* b, const float* b_lo, float* c, int m, int n, int k, void* stream);
/* Tensor-core kernel variants for A/B tests (1 on, 0 off, -1 unchanged): CTA
 * pairs (cta_group::2), persistent multi-wave kernels, cluster split-K. */
int rgb_set_tc_config(int pair, int persist, int csplit);
/* Tensor-core GEMM precision (the north_star's separately bounded TF32 mode;
 * the reference is float64 throughout, kernels.py:84-103): 3 (default) =
 * 3xTF32, fp32-exact (hi*hi + hi*lo + lo*hi per k-step); 1 = plain TF32
 * (hi*hi only, ~1e-3 relative per product; bound in tests/test_gpu_engine.py).
 * Affects only the tcgen05 GEMMs; SIMT and SCC kernels stay fp32.  Read at
 * launch time, so CUDA graphs captured before a change keep the old mode. */
int rgb_set_tc_precision(int terms);

/* Instrumentation (no reference counterpart; the reference times whole
 * iterations with perf_counter, engine.py:733-758).  rgb_launch_count: kernel
 * launches issued by this library since load.  When profiling is enabled
 * every launch is bracketed by CUDA events on its stream; collect()
 * synchronises and accumulates device time, algorithmic FLOPs and bytes per
 * category (0 ew, 1 hoisted gemm, 2 per-frame gemm, 3 per-frame ew, 4 dW,
 * 5 softmax, 6 inject, 7 sgd, 8 transpose, 9 persistent SCC). */
int rgb_launch_count(int64_t* n);
int rgb_profile_enable(int on);
int rgb_profile_collect(void);
int rgb_profile_reset(void);
int rgb_profile_read(int category, double* ms, int64_t* launches, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* RNNGRAPH_B200_H */
