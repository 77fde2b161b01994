/*
 * lfmmi.h — C-ABI of the B200-native LF-MMI hot path (libpaper_lfmmi.so).
 *
 * Plain pointers and sizes only: no torch, no C++ types.  Every device
 * pointer is a CUDA global-memory address on the current device; `stream`
 * is a cudaStream_t passed as void*.  Entry points return LFMMI_OK (0) or a
 * nonzero status; lfmmi_last_error() returns a thread-local message.
 *
 * Reference interfaces replaced (chainloss 0.1.0, /root/reference/pkg/src/chainloss):
 *   lfmmi_graphs_create      graph.py:216-301   ChainGraphBatch._build (+ device residency)
 *   lfmmi_forward_backward   forward_backward.py:290-307  forward_backward (fused, no trellis)
 *   lfmmi_chain_loss         loss.py:42-84      chain_loss (num + den + combination)
 *   lfmmi_forward_kernel     _kernels.py:54-122   forward_kernel   (parity/debug seam)
 *   lfmmi_backward_kernel    _kernels.py:125-191  backward_kernel  (parity/debug seam)
 *   lfmmi_posterior_kernel   _kernels.py:194-224  posterior_kernel (parity/debug seam)
 *
 * Semantics are those of the reference: scaled probability-
 * space recursion with leaky HMM, finals applied at each item's own last
 * frame, per-item numerical failure reported as data (fail frame >= 0, NaN
 * log-probability, zero posterior rows), never as an error status.
 */
#ifndef LFMMI_H_
#define LFMMI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFMMI_OK 0
#define LFMMI_ERR_INVALID 1     /* bad argument / shape (reference: ValueError) */
#define LFMMI_ERR_CUDA 2        /* CUDA runtime error */
#define LFMMI_ERR_UNSUPPORTED 3 /* graph too large for the on-chip path, etc. */

#define LFMMI_F32 0
#define LFMMI_F64 1

#define LFMMI_POST_WRITE 0    /* posteriors[b,t,:]  = gamma                     */
#define LFMMI_POST_SUBTRACT 1 /* posteriors[b,t,:] -= gamma                     */
#define LFMMI_POST_ADD 2      /* posteriors[b,t,:] += gamma  (grad = num - den) */
#define LFMMI_POST_NEGATE 3   /* posteriors[b,t,:]  = -gamma                    */

typedef struct lfmmi_graphs lfmmi_graphs;

/* Message describing the last nonzero status returned on this thread. */
const char *lfmmi_last_error(void);

/*
 * Process-wide dispatch / debug options, one struct parsed once from the
 * LFMMI_OPTIONS environment variable ("name=value,...") and changeable here.
 * Names:
 *   tile, stream, linear   0/1: kernel families the dispatcher may use
 *   linear_split           numerators as forward | backward warps
 *   linear_k16w            warps per direction for numerators with S > 256 (2 or 1)
 *   linear_k16             1: one numerator launch for every K
 *   emit                   emissions pre-pass of the chain loss (1 auto: skipped for
 *                          dens whose arc pack exceeds shared memory; 2 always; 0 never)
 *   split                  den split kernel: -1 auto / 0 off / 1 force
 *   split_clusters, split_h64   cluster count (0 auto), midpoint in 64ths of T
 *   small_arcs, small_indeg     graphs with <= 512 states, <= small_arcs arcs and
 *                          in-degree <= small_indeg take the numerator-sized kernels
 *   tile_g                 tile-pack lanes per state (0 auto; pack time)
 *   tile_xdb, tile_persist den tile kernel: double-buffered slots; persistent CTAs
 *                          over an in-kernel LPT when B > SMs (0 off, 1 auto, >= 2 force)
 *   stream_mode            "auto", "split", "1024x1", "1024x2", "512x2"
 *   stream_ring            TMA slot ring of the 1024x1 / 1024x2 stream kernels
 *   ssplit_ring            ... of the stream split kernel (default off)
 *   num_group              threads per utterance of the generic numerator kernel
 *   serial                 -1 auto / 0 / 1: numerator pass before the den pass
 *   sched_iters, chore_bias     pack-time scheduling knobs
 *   debug, profile         stderr notes; "", "split", "tile" cycle counters
 * Unknown names return LFMMI_ERR_INVALID.  Not thread-safe against
 * concurrent launches: set them before use.
 */
int lfmmi_set_option(const char *name, const char *value);
int lfmmi_get_option(const char *name, char *buf, size_t len);
int lfmmi_reset_options(void);

/* Library version string. */
const char *lfmmi_version(void);

/*
 * Number of kernels the last successful lfmmi_chain_loss call on this thread
 * launched (1 = fused single-launch path, 3 = two-pass path: denominator,
 * numerators, gradient combine + batch totals).  Diagnostic.
 */
int32_t lfmmi_last_launch_count(void);

/*
 * Name of the kernel that ran the last forward-backward pass launched on this
 * thread, e.g. "fb_split_kernel ..." for a WSJ-sized denominator.  Diagnostic
 * (benchmarks label their roofline line with it).
 */
const char *lfmmi_last_den_kernel(void);

/* Name of the kernel of the last forward-backward launch of any graph size on
 * this thread (numerator passes included, e.g. "fb_linear_kernel<4>"). */
const char *lfmmi_last_kernel(void);

/*
 * Build a device-resident graph batch from the reference's padded host
 * layout (graph.py:253-279).  G physical rows; row r has row_num_states[r]
 * states and row_num_arcs[r] arcs.  Arrays are (G, max_arcs) in the
 * from-state-sorted ("forward_*") layout and, optionally, the to-state-sorted
 * ("backward_*") layout.  If the backward arrays are NULL they are derived by
 * a stable sort.  final_probs is (G, max_states), initial_states is (G).
 * Graph data is uploaded once (synchronously) and stays resident until
 * lfmmi_graphs_destroy.
 */
int lfmmi_graphs_create(int32_t num_rows, int32_t max_states, int32_t max_arcs, int32_t num_pdfs,
                        const int64_t *row_num_states, const int64_t *row_num_arcs,
                        const uint32_t *fw_from, const uint32_t *fw_to, const uint32_t *fw_pdf,
                        const double *fw_prob, const uint32_t *bw_from, const uint32_t *bw_to,
                        const uint32_t *bw_pdf, const double *bw_prob, const double *final_probs,
                        const uint32_t *initial_states, lfmmi_graphs **out);

/*
 * Graph batch of LINEAR CHAINS from caller-owned DEVICE arrays: no copy, no
 * allocation, no synchronisation — a training step assembles it from cached
 * per-utterance records with one async H2D copy.  A linear chain has only
 * self-loops s -> s and entry arcs s-1 -> s, at most one of each per state
 * (the reference's numerators: toy_builder.py:218-265 build_numerator).
 *   items   (num_rows x 4) int32: state offset into `states`, S, initial state, 0
 *   states  (sum S x 4)  u32 per state: fp32 bits of the self-loop prob (0 if
 *           none), fp32 bits of the entry-arc prob (0 if none), self pdf |
 *           entry pdf << 16, fp32 bits of the final prob
 * max_states <= 512, num_pdfs <= 65536.  The arrays must outlive the handle
 * and every launch that uses it; lfmmi_graphs_destroy frees only the handle.
 * Such a handle is usable by the fp32 paths with the uniform leak only.
 * (lfmmi_graphs_create builds the same records itself when every row of a
 * host batch is a linear chain.)
 */
int lfmmi_graphs_create_linear(int32_t num_rows, int32_t max_states, int32_t num_pdfs,
                               const int32_t *items, const uint32_t *states, lfmmi_graphs **out);

int lfmmi_graphs_destroy(lfmmi_graphs *graphs);

/* Shape queries on a graph handle. */
int lfmmi_graphs_info(const lfmmi_graphs *graphs, int32_t *num_rows, int32_t *max_states,
                      int32_t *max_arcs, int32_t *num_pdfs);

/*
 * Bytes of caller-provided device workspace needed by lfmmi_forward_backward
 * / lfmmi_chain_loss for a batch of `total_frames` = sum of lengths over
 * graph batches whose largest state count is `max_states`.
 */
size_t lfmmi_workspace_size(int32_t max_states, int64_t total_frames, int32_t precision);

/*
 * Fused forward-backward + posteriors for one graph batch (one launch).
 *   row_map      (B)        int64  item -> physical graph row      [device]
 *   loglikes     (B,T,D)    f32/f64 network outputs (log domain)   [device]
 *   lengths      (B)        int32  valid frames per item (>= 1)    [device]
 *   leak_pi      (G,S_max)  f32/f64 custom leak distribution, or NULL for uniform 1/S_g
 *   total_frames an upper bound on sum(lengths) (e.g. B * T_max); sizes the ragged trellis
 *   workspace    device scratch of >= lfmmi_workspace_size(S_max, total_frames, precision) bytes
 *   posteriors   (B,T,D)    f32/f64  written per `post_mode`; rows of failed items
 *                           are set to zero in every mode; padded rows are zeroed
 *                           by the writing modes (WRITE, NEGATE)
 *   other_fail   (B) int32 or NULL: items whose other-graph recursion failed get
 *                zero rows (used for the second pass of chain_loss)
 *   log_probs    (B) f64 out (NaN when failed); fail_frames (B) int32 out (-1 or frame)
 *   scale_logs   (B,T) f64 out or NULL
 * precision selects f32 (LFMMI_F32) or f64 (LFMMI_F64) for all real arrays.
 */
int lfmmi_forward_backward(const lfmmi_graphs *graphs, const int64_t *row_map, int32_t batch,
                           int32_t max_frames, int32_t num_pdfs, int32_t precision,
                           const void *loglikes, const int32_t *lengths, double leak,
                           double scale_floor, const void *leak_pi, int64_t total_frames,
                           void *workspace, size_t workspace_bytes, void *posteriors,
                           int32_t post_mode,
                           const int32_t *other_fail, double *log_probs, int32_t *fail_frames,
                           double *scale_logs, void *stream);

/*
 * Ragged ("packed") variant: loglikes / posteriors are (sum_b T_b, D) with item
 * b's frames at rows [sum_{j<b} T_j, sum_{j<=b} T_j) — no padding, any length
 * order (device-side batching; replaces the host
 * make_batch sort + zero-pad, batching.py:52-97).  max_frames = max_b T_b.
 */
int lfmmi_forward_backward_packed(const lfmmi_graphs *graphs, const int64_t *row_map,
                                  int32_t batch, int32_t max_frames, int32_t num_pdfs,
                                  int32_t precision, const void *loglikes, const int32_t *lengths,
                                  double leak, double scale_floor, const void *leak_pi,
                                  int64_t total_frames, void *workspace, size_t workspace_bytes,
                                  void *posteriors, int32_t post_mode, const int32_t *other_fail,
                                  double *log_probs, int32_t *fail_frames, double *scale_logs,
                                  void *stream);

/* Workspace bytes for lfmmi_chain_loss (both trellises + numerator posteriors). */
size_t lfmmi_chain_loss_workspace_size(const lfmmi_graphs *numerators,
                                       const lfmmi_graphs *denominator, int32_t batch,
                                       int32_t max_frames, int32_t num_pdfs,
                                       int64_t total_frames, int32_t precision);

/*
 * LF-MMI objective and gradient for one batch (loss.py:42-84).  The numerator
 * pass (posteriors into the workspace) runs on an internal auxiliary stream
 * concurrently with the denominator pass (grad = -gamma_den); a combine step
 * adds gamma_num and zeroes rows of items where either recursion failed
 * (loss.py:61-69), then a reduction writes
 * totals[0] = sum_ok(num_lp - den_lp), totals[1] = sum_ok(T_b),
 * totals[2] = #failed   (device f64[3]; sum-reducible across ranks).
 * All work is ordered after prior work on `stream` and before later work on it.
 */
int lfmmi_chain_loss(const lfmmi_graphs *numerators, const int64_t *num_row_map,
                     const lfmmi_graphs *denominator, const int64_t *den_row_map, int32_t batch,
                     int32_t max_frames, int32_t num_pdfs, int32_t precision,
                     const void *loglikes, const int32_t *lengths, double leak,
                     double scale_floor, const void *num_leak_pi, const void *den_leak_pi,
                     int64_t total_frames, void *workspace, size_t workspace_bytes, void *grad,
                     double *num_log_probs,
                     double *den_log_probs, int32_t *num_fail, int32_t *den_fail,
                     double *totals, void *stream);

/*
 * Native text-FST ingestion (host only; no GPU needed).  Format and error
 * contract of fst_io.py:53-110 (arc "src dst label [weight]", label = pdf+1,
 * final "state [weight]", weight = -ln p, '#' comments, states densely
 * re-indexed by first appearance; errors carry 1-based line numbers in
 * lfmmi_last_error()).  Call _size first, then _parse into caller arrays
 * (num_arcs entries each; final_probs has num_states entries, 0 = not final).
 * Replaces: fst_io.py:53 parse_fst_text.
 */
int lfmmi_fst_text_size(const char *text, size_t length, int32_t num_pdfs,
                        int64_t *num_states, int64_t *num_arcs);
int lfmmi_fst_text_parse(const char *text, size_t length, int32_t num_pdfs, int64_t num_states,
                         int64_t num_arcs, uint32_t *src, uint32_t *dst, uint32_t *pdf,
                         double *prob, double *final_probs);

/* Ragged variant of lfmmi_chain_loss (loglikes / grad are (sum_b T_b, D)). */
int lfmmi_chain_loss_packed(const lfmmi_graphs *numerators, const int64_t *num_row_map,
                            const lfmmi_graphs *denominator, const int64_t *den_row_map,
                            int32_t batch, int32_t max_frames, int32_t num_pdfs, int32_t precision,
                            const void *loglikes, const int32_t *lengths, double leak,
                            double scale_floor, const void *num_leak_pi, const void *den_leak_pi,
                            int64_t total_frames, void *workspace, size_t workspace_bytes,
                            void *grad, double *num_log_probs, double *den_log_probs,
                            int32_t *num_fail, int32_t *den_fail, double *totals, void *stream);

/*
 * Parity/debug seam mirroring the numba kernels argument-for-argument (f64,
 * caller-allocated outputs written in place, trellis layouts (B,T+1,S_max)).
 * `expl` is the shifted emission probability array (B,T,D) f64.
 */
int lfmmi_forward_kernel(const lfmmi_graphs *graphs, const int64_t *row_map, int32_t batch,
                         int32_t max_frames, int32_t num_pdfs, const double *expl,
                         const int32_t *lengths, double leak, const double *leak_pi,
                         double scale_floor, double *alpha, double *scales,
                         int64_t *fail_frames, void *stream);

int lfmmi_backward_kernel(const lfmmi_graphs *graphs, const int64_t *row_map, int32_t batch,
                          int32_t max_frames, int32_t num_pdfs, const double *expl,
                          const int32_t *lengths, const double *scales, double leak,
                          const double *leak_pi, const int64_t *fail_frames, double *beta,
                          void *stream);

int lfmmi_posterior_kernel(const lfmmi_graphs *graphs, const int64_t *row_map, int32_t batch,
                           int32_t max_frames, int32_t num_pdfs, const double *expl,
                           const int32_t *lengths, const double *alpha, const double *beta,
                           const int64_t *fail_frames, double *gamma, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* LFMMI_H_ */
