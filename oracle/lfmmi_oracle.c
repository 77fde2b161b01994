/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference LF-MMI
 * recursions, used as the parity checker for the CUDA path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path never calls it.
 *
 * Parity status: pinned.  tests/test_oracle_golden.py checks these functions
 * bit-for-bit against golden vectors produced by the reference implementation
 * itself (tests/golden/make_golden.py imports chainloss 0.1.0 from
 * /root/reference/pkg/src and records its outputs).
 *
 * Each function is a sequential fp64 transliteration of one numba kernel in
 * /root/reference/pkg/src/chainloss/_kernels.py with the same operation order
 * (per-state accumulation in CSR order, column totals summed in state order),
 * so results agree with the reference bit for bit when compiled with
 * -ffp-contract=off.
 *
 * Array conventions are exactly those of the numba kernels:
 *   expl      (B, T, D) f64      shifted emission probabilities
 *   lengths   (B)       i64      non-increasing
 *   bvalid    (T)       i64      valid batch size per step
 *   row_map   (B)       i64      item -> physical graph row
 *   *_from/_to/_pdf (G, I) u32, *_prob (G, I) f64, *_index (G, S, 2) u32
 *   final     (G, S) f64, init (G) u32, leak_pi (G, S) f64
 *   alpha/beta (B, T+1, S) f64, scales (B, T) f64, fail (B) i64
 */
#include <math.h>
#include <stdint.h>

#define A3(arr, i, j, k, n1, n2) (arr)[((int64_t)(i) * (n1) + (j)) * (n2) + (k)]

/* cl/_kernels.py:54-122 forward_kernel */
void oracle_forward(const double *expl, const int64_t *lengths, const int64_t *bvalid,
                    const int64_t *row_map, const uint32_t *bw_from, const uint32_t *bw_pdf,
                    const double *bw_prob, const uint32_t *bw_index, const double *final_probs,
                    const uint32_t *init_states, double leak, const double *leak_pi,
                    double scale_floor, int64_t batch, int64_t t_max, int64_t num_pdfs,
                    int64_t g_rows, int64_t i_max, int64_t n_states, double *alpha,
                    double *scales, int64_t *fail_frames) {
    (void)g_rows;
    const int64_t T1 = t_max + 1;
    for (int64_t b = 0; b < batch; ++b)                       /* :76-77 */
        A3(alpha, b, 0, init_states[row_map[b]], T1, n_states) = 1.0;

    for (int64_t t = 1; t <= t_max; ++t) {                    /* :79 */
        const int64_t active = bvalid[t - 1];
        for (int64_t b = 0; b < active; ++b) {                /* :82-99 */
            if (fail_frames[b] >= 0) continue;
            const int64_t g = row_map[b];
            for (int64_t s = 0; s < n_states; ++s) {
                const uint32_t lo = bw_index[(g * n_states + s) * 2 + 0];
                const uint32_t hi = bw_index[(g * n_states + s) * 2 + 1];
                double acc = 0.0;
                for (uint32_t i = lo; i < hi; ++i) {
                    acc += bw_prob[g * i_max + i] *
                           A3(alpha, b, t - 1, bw_from[g * i_max + i], T1, n_states) *
                           A3(expl, b, t - 1, bw_pdf[g * i_max + i], t_max, num_pdfs);
                }
                if (t == lengths[b]) acc *= final_probs[g * n_states + s];
                A3(alpha, b, t, s, T1, n_states) = acc;
            }
        }
        for (int64_t b = 0; b < active; ++b) {                /* :101-122 */
            if (fail_frames[b] >= 0) continue;
            const int64_t g = row_map[b];
            double *col = &A3(alpha, b, t, 0, T1, n_states);
            double total = 0.0;
            for (int64_t s = 0; s < n_states; ++s) total += col[s];
            if (leak > 0.0 && total > 0.0) {
                for (int64_t s = 0; s < n_states; ++s)
                    col[s] += leak * leak_pi[g * n_states + s] * total;
                total = 0.0;
                for (int64_t s = 0; s < n_states; ++s) total += col[s];
            }
            if (!(total >= scale_floor) || total == INFINITY) {
                fail_frames[b] = t - 1;
                for (int64_t s = 0; s < n_states; ++s) col[s] = 0.0;
                continue;
            }
            const double inv = 1.0 / total;
            for (int64_t s = 0; s < n_states; ++s) col[s] *= inv;
            scales[b * t_max + t - 1] = total;
        }
    }
}

/* cl/_kernels.py:125-191 backward_kernel */
void oracle_backward(const double *expl, const int64_t *lengths, const int64_t *bvalid,
                     const int64_t *row_map, const uint32_t *fw_to, const uint32_t *fw_pdf,
                     const double *fw_prob, const uint32_t *fw_index, const double *final_probs,
                     const double *scales, double leak, const double *leak_pi,
                     const int64_t *fail_frames, int64_t batch, int64_t t_max, int64_t num_pdfs,
                     int64_t g_rows, int64_t i_max, int64_t n_states, double *beta) {
    (void)g_rows; (void)batch;
    const int64_t T1 = t_max + 1;
    for (int64_t t = t_max; t >= 1; --t) {
        const int64_t active = bvalid[t - 1];
        for (int64_t b = 0; b < active; ++b) {                /* :152-158 */
            if (fail_frames[b] >= 0 || lengths[b] != t) continue;
            const int64_t g = row_map[b];
            const double factor = (1.0 + leak) / scales[b * t_max + t - 1];
            for (int64_t s = 0; s < n_states; ++s)
                A3(beta, b, t, s, T1, n_states) = final_probs[g * n_states + s] * factor;
        }
        for (int64_t b = 0; b < active; ++b) {                /* :160-175 */
            if (fail_frames[b] >= 0) continue;
            const int64_t g = row_map[b];
            for (int64_t s = 0; s < n_states; ++s) {
                const uint32_t lo = fw_index[(g * n_states + s) * 2 + 0];
                const uint32_t hi = fw_index[(g * n_states + s) * 2 + 1];
                double acc = 0.0;
                for (uint32_t i = lo; i < hi; ++i) {
                    acc += fw_prob[g * i_max + i] *
                           A3(expl, b, t - 1, fw_pdf[g * i_max + i], t_max, num_pdfs) *
                           A3(beta, b, t, fw_to[g * i_max + i], T1, n_states);
                }
                A3(beta, b, t - 1, s, T1, n_states) = acc;
            }
        }
        if (t - 1 >= 1) {                                     /* :177-191 */
            for (int64_t b = 0; b < active; ++b) {
                if (fail_frames[b] >= 0) continue;
                const int64_t g = row_map[b];
                double *col = &A3(beta, b, t - 1, 0, T1, n_states);
                if (leak > 0.0) {
                    double dot = 0.0;
                    for (int64_t s = 0; s < n_states; ++s) dot += leak_pi[g * n_states + s] * col[s];
                    const double add = leak * dot;
                    for (int64_t s = 0; s < n_states; ++s) col[s] += add;
                }
                const double inv = 1.0 / scales[b * t_max + t - 2];
                for (int64_t s = 0; s < n_states; ++s) col[s] *= inv;
            }
        }
    }
}

/* cl/_kernels.py:194-224 posterior_kernel */
void oracle_posterior(const double *expl, const int64_t *lengths, const int64_t *row_map,
                      const int64_t *item_ntrans, const uint32_t *fw_from, const uint32_t *fw_to,
                      const uint32_t *fw_pdf, const double *fw_prob, const double *alpha,
                      const double *beta, const int64_t *fail_frames, int64_t batch,
                      int64_t t_max, int64_t num_pdfs, int64_t i_max, int64_t n_states,
                      double *gamma) {
    const int64_t T1 = t_max + 1;
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t t = 0; t < t_max; ++t) {
            if (t >= lengths[b] || fail_frames[b] >= 0) continue;
            const int64_t g = row_map[b];
            for (int64_t i = 0; i < item_ntrans[b]; ++i) {
                const uint32_t d = fw_pdf[g * i_max + i];
                A3(gamma, b, t, d, t_max, num_pdfs) +=
                    A3(alpha, b, t, fw_from[g * i_max + i], T1, n_states) * fw_prob[g * i_max + i] *
                    A3(expl, b, t, d, t_max, num_pdfs) *
                    A3(beta, b, t + 1, fw_to[g * i_max + i], T1, n_states);
            }
        }
    }
}
