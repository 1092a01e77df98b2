/* Plain-C restatement of the reference numeric kernels.  TEST ORACLE ONLY.
 *
 * Restates /root/reference/pkg/src/balsim/_kernels/_compiled.pyx:11-86 (and the
 * pure twin _pure.py:11-105) with the same integer widths (long long) and the
 * same floating-point expression order, so results are bit-identical.  Built
 * with -ffp-contract=off so gcc cannot fuse the multiply-divide chains.
 */
#include <stdint.h>

/* _compiled.pyx:11-17 */
long long orc_sum_pair_counts(const long long* len, long long n) {
    long long total = 0;
    for (long long i = 0; i < n; ++i) total += len[i] * (len[i] + 1) / 2;
    return total;
}

/* _compiled.pyx:20-27 */
long long orc_range_pair_sum(const long long* s, const long long* e, long long n) {
    long long total = 0;
    for (long long i = 0; i < n; ++i) total += (e[i] * (e[i] + 1) - s[i] * (s[i] + 1)) / 2;
    return total;
}

/* _compiled.pyx:30-47 */
double orc_kernel_latency_sum(const long long* q, const long long* kv, long long n,
                              long long tile, const long long* cq, const double* cv,
                              long long ncurve, double op_scale) {
    double total = 0.0;
    for (long long i = 0; i < n; ++i) {
        if (q[i] == 0) continue;
        long long j = ncurve - 1;
        while (j > 0 && cq[j] > q[i]) --j;
        long long padded = ((q[i] + tile - 1) / tile) * tile;
        double x = op_scale * (double)(padded * kv[i]);
        total += x / cv[j];
    }
    return total;
}

/* _compiled.pyx:50-86: longest-first min-W placement; -1 = unplaceable. */
void orc_heuristic_fill(const long long* len, long long n, int n_mb, long long l_max,
                        double attn_coeff, double linear_coeff,
                        long long* bin_len, long long* bin_pairs, int* out) {
    for (int j = 0; j < n_mb; ++j) { bin_len[j] = 0; bin_pairs[j] = 0; }
    for (long long i = 0; i < n; ++i) {
        long long d = len[i];
        int w_idx = 0;
        double best = attn_coeff * (double)bin_pairs[0] + linear_coeff * (double)bin_len[0];
        for (int j = 1; j < n_mb; ++j) {
            double w = attn_coeff * (double)bin_pairs[j] + linear_coeff * (double)bin_len[j];
            if (w < best) { best = w; w_idx = j; }
        }
        int target;
        if (bin_len[w_idx] + d <= l_max) {
            target = w_idx;
        } else {
            int l_idx = 0;
            for (int j = 1; j < n_mb; ++j)
                if (bin_len[j] < bin_len[l_idx]) l_idx = j;
            if (bin_len[l_idx] + d <= l_max) target = l_idx;
            else { out[i] = -1; continue; }
        }
        bin_len[target] += d;
        bin_pairs[target] += d * (d + 1) / 2;
        out[i] = target;
    }
}
