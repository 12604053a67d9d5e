/*
 * ORACLE — test infrastructure only.  Nothing in the product path
 * (paper_2504_08850_b200/) may link, load or call this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 *
 * Plain-C restatement of the reference's strict float32 arithmetic contract:
 *
 *   matmul_f32: C[i,c] = sum_k fl(A[i,k] * B[k,c]), k ascending, one rounding
 *               per product and one per add, no FMA contraction.
 *               Follows /root/reference/pkg/src/specexit/kernels/_ckern.pyx:16-31
 *               (the i, k, c loop order) and kernels/_py.py:11-16.
 *   seq_sum_f32: out[i] = ((x[i,0] + x[i,1]) + ...) from 0, left to right.
 *               Follows kernels/_ckern.pyx:34-46 and kernels/_py.py:19-24.
 *
 * Compiled with -O2 -ffp-contract=off (oracle/Makefile), as the reference's
 * setup.py:17-24 compiles its Cython kernel.
 */
#include <stdint.h>
#include <string.h>

void oracle_matmul_f32(const float *a, const float *b, float *out,
                       int64_t m, int64_t k, int64_t n) {
    memset(out, 0, (size_t)(m * n) * sizeof(float));
    for (int64_t i = 0; i < m; ++i) {
        float *o = out + i * n;
        for (int64_t j = 0; j < k; ++j) {
            const float aik = a[i * k + j];
            const float *bj = b + j * n;
            for (int64_t c = 0; c < n; ++c) {
                float p = aik * bj[c];
                o[c] = o[c] + p;
            }
        }
    }
}

/* Column-gathered variant of matmul_f32 for a single row: out[c] =
 * sum_j fl(h[j] * W[j, ids[c]]) with W stored (k, ld) row-major.  Same
 * operation sequence as matmul_f32(h, ascontiguousarray(W[:, ids])), i.e.
 * reference model.py:313-314, without materialising the gathered copy. */
void oracle_gather_dot_f32(const float *h, const float *w, int64_t ld,
                           const int64_t *ids, int64_t nids, int64_t k,
                           float *out) {
    for (int64_t c = 0; c < nids; ++c) out[c] = 0.0f;
    for (int64_t j = 0; j < k; ++j) {
        const float hj = h[j];
        const float *wj = w + j * ld;
        for (int64_t c = 0; c < nids; ++c) {
            float p = hj * wj[ids[c]];
            out[c] = out[c] + p;
        }
    }
}

void oracle_seq_sum_f32(const float *x, float *out, int64_t m, int64_t n) {
    for (int64_t i = 0; i < m; ++i) {
        float acc = 0.0f;
        for (int64_t j = 0; j < n; ++j) acc = acc + x[i * n + j];
        out[i] = acc;
    }
}
