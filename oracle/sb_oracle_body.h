/* Body of the CPU oracle, instantiated once per precision by sb_oracle.c.
 *
 * TEST INFRASTRUCTURE ONLY: this restates the reference's tiled NumPy kernels
 * so tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can check
 * the CUDA path. Nothing in the product links or calls it.
 *
 * Expects REAL (double|float), SFX (token), EXP, LOG1P, SQRT to be defined.
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)

/* numerics.py:19 (threshold 15.0) and numerics.py:33-47 (softplus_stable):
 * log1p(exp(min(x, 15))) for x <= 15, else x itself. */
static inline REAL FN(sbo_softplus_)(REAL x) {
    if (x <= (REAL)15.0) return LOG1P(EXP(x));
    return x;
}

/* One recomputed tile, shared by the forward and both backward phases:
 * blocked.py:177-186 (forward) and blocked.py:325-335 (recompute_tile).
 * z[r][c] = q_r . k_c * scale; lt = -softplus(z), zeroed where masked;
 * A = exp(z + suffix_cumsum(lt) + acc[r]) on the mask, 0 elsewhere.
 * The diagonal mask keeps key column c < query row r (blocked.py:110-112). */
static void FN(sbo_tile_)(const REAL* q, const REAL* k, int d, int rows, int cols,
                          int diag, REAL scale, const REAL* acc,
                          REAL* z, REAL* lt, REAL* A) {
    for (int r = 0; r < rows; ++r) {
        for (int c = 0; c < cols; ++c) {
            const REAL* qr = q + (size_t)r * d;
            const REAL* kc = k + (size_t)c * d;
            REAL s = 0;
#pragma omp simd reduction(+ : s)
            for (int e = 0; e < d; ++e) s += qr[e] * kc[e];
            z[r * cols + c] = s * scale;
        }
        for (int c = 0; c < cols; ++c) {
            int masked = diag && !(c < r);
            lt[r * cols + c] = masked ? (REAL)0 : -FN(sbo_softplus_)(z[r * cols + c]);
        }
        /* _cumsum_left (blocked.py:209-211): inclusive suffix sums, summed
         * sequentially from the right edge like np.cumsum on the flipped row */
        REAL cum = 0;
        for (int c = cols - 1; c >= 0; --c) {
            cum += lt[r * cols + c];
            int masked = diag && !(c < r);
            A[r * cols + c] = masked ? (REAL)0 : EXP(z[r * cols + c] + cum + acc[r]);
        }
    }
}

/* blocked_forward (blocked.py:129-206) with two_phase=True: per query block,
 * key blocks right to left, optional skip (blocked.py:175-176), M snapshots
 * (blocked.py:188-189).  M is laid out [tile(qb,kb)][block] with
 * tile(qb,kb) = qb*(qb+1)/2 + kb.  Returns visited tile count. */
long long FN(sbo_forward_)(int L, int d, int block, const REAL* q, const REAL* k,
                           const REAL* v, int skip, double skip_eps, REAL* o,
                           REAL* a_out, int64_t* first_kb, REAL* M) {
    if (L < 1 || block < 1 || d < 1) return -1;
    if (skip && !(skip_eps > 0.0 && skip_eps < 1.0)) return -2;
    const int nb = (L + block - 1) / block;
    const REAL scale = (REAL)(1.0 / sqrt((double)d));
    /* NumPy 2 (NEP 50): a_cur.max() < python-float compares in the array dtype */
    const REAL log_eps = (REAL)log(skip_eps > 0 ? skip_eps : 0.5);
    REAL* z = (REAL*)malloc(sizeof(REAL) * block * block);
    REAL* lt = (REAL*)malloc(sizeof(REAL) * block * block);
    REAL* A = (REAL*)malloc(sizeof(REAL) * block * block);
    REAL* a_cur = (REAL*)malloc(sizeof(REAL) * block);
    long long visited = 0;
    memset(o, 0, sizeof(REAL) * (size_t)L * d);
    for (int qb = 0; qb < nb; ++qb) {
        const int qs = qb * block, qe = qs + block < L ? qs + block : L, rows = qe - qs;
        for (int r = 0; r < rows; ++r) a_cur[r] = 0;
        int lowest = qb;
        for (int kb = qb; kb >= 0; --kb) {
            if (skip && kb < qb) {
                REAL mx = a_cur[0];
                for (int r = 1; r < rows; ++r) mx = a_cur[r] > mx ? a_cur[r] : mx;
                if (mx < log_eps) break;
            }
            const int ks = kb * block, ke = ks + block < L ? ks + block : L, cols = ke - ks;
            FN(sbo_tile_)(q + (size_t)qs * d, k + (size_t)ks * d, d, rows, cols, kb == qb,
                          scale, a_cur, z, lt, A);
            for (int r = 0; r < rows; ++r) {
                REAL* orow = o + (size_t)(qs + r) * d;
                for (int c = 0; c < cols; ++c) {
                    const REAL w = A[r * cols + c];
                    const REAL* vc = v + (size_t)(ks + c) * d;
#pragma omp simd
                    for (int e = 0; e < d; ++e) orow[e] += w * vc[e];
                }
            }
            if (M) {
                REAL* m = M + ((size_t)qb * (qb + 1) / 2 + kb) * block;
                for (int r = 0; r < rows; ++r) m[r] = a_cur[r];
            }
            for (int r = 0; r < rows; ++r) {
                REAL s = 0;
                for (int c = 0; c < cols; ++c) s += lt[r * cols + c];
                a_cur[r] = a_cur[r] + s;
            }
            ++visited;
            lowest = kb;
        }
        for (int r = 0; r < rows; ++r) a_out[qs + r] = a_cur[r];
        first_kb[qb] = lowest;
    }
    free(z); free(lt); free(A); free(a_cur);
    return visited;
}

/* dZ for one tile given the running b in effect (blocked.py:347-352,
 * blocked.py:378-383): dW = dO V^T - row_offset; dAt = A*dW;
 * sigma = 1 - exp(lt); dZ = dAt - sigma*(prefix_cumsum(dAt) + b). */
static void FN(sbo_dz_)(const REAL* dob, const REAL* vb, int d, int rows, int cols,
                        const REAL* off, const REAL* A, const REAL* lt, const REAL* b,
                        REAL* dAt, REAL* dZ) {
    for (int r = 0; r < rows; ++r) {
        for (int c = 0; c < cols; ++c) {
            const REAL* dr = dob + (size_t)r * d;
            const REAL* vc = vb + (size_t)c * d;
            REAL s = 0;
#pragma omp simd reduction(+ : s)
            for (int e = 0; e < d; ++e) s += dr[e] * vc[e];
            if (off) s = s - off[r];
            dAt[r * cols + c] = A[r * cols + c] * s;
        }
        REAL pfx = 0;
        for (int c = 0; c < cols; ++c) {
            pfx += dAt[r * cols + c];
            const REAL sig = (REAL)1.0 - EXP(lt[r * cols + c]);
            dZ[r * cols + c] = dAt[r * cols + c] - sig * (pfx + b[r]);
        }
    }
}

/* blocked_backward_twophase (blocked.py:299-392). Phase 1: per query block,
 * key blocks first_kb..qb left to right, stores N (b in effect), dQ.
 * Phase 2: per key block, query blocks top to bottom over visited tiles,
 * dK and dV.  N has M's layout. */
int FN(sbo_backward_twophase_)(int L, int d, int block, const REAL* q, const REAL* k,
                               const REAL* v, const REAL* d_o, const REAL* row_offset,
                               const int64_t* first_kb, const REAL* M, REAL* N,
                               REAL* dq, REAL* dk, REAL* dv) {
    if (L < 1 || block < 1 || d < 1) return -1;
    const int nb = (L + block - 1) / block;
    const REAL scale = (REAL)(1.0 / sqrt((double)d));
    const size_t tb = (size_t)block * block;
    REAL *z = (REAL*)malloc(sizeof(REAL) * tb), *lt = (REAL*)malloc(sizeof(REAL) * tb);
    REAL *A = (REAL*)malloc(sizeof(REAL) * tb), *dAt = (REAL*)malloc(sizeof(REAL) * tb);
    REAL *dZ = (REAL*)malloc(sizeof(REAL) * tb), *b = (REAL*)malloc(sizeof(REAL) * block);
    REAL *acc = (REAL*)malloc(sizeof(REAL) * d);
    REAL *tk = (REAL*)malloc(sizeof(REAL) * (size_t)block * d);
    REAL *tv = (REAL*)malloc(sizeof(REAL) * (size_t)block * d);
    memset(dq, 0, sizeof(REAL) * (size_t)L * d);
    memset(dk, 0, sizeof(REAL) * (size_t)L * d);
    memset(dv, 0, sizeof(REAL) * (size_t)L * d);
    for (int qb = 0; qb < nb; ++qb) {
        const int qs = qb * block, qe = qs + block < L ? qs + block : L, rows = qe - qs;
        for (int r = 0; r < rows; ++r) b[r] = 0;
        for (int kb = (int)first_kb[qb]; kb <= qb; ++kb) {
            const int ks = kb * block, ke = ks + block < L ? ks + block : L, cols = ke - ks;
            const size_t t = (size_t)qb * (qb + 1) / 2 + kb;
            FN(sbo_tile_)(q + (size_t)qs * d, k + (size_t)ks * d, d, rows, cols, kb == qb,
                          scale, M + t * block, z, lt, A);
            FN(sbo_dz_)(d_o + (size_t)qs * d, v + (size_t)ks * d, d, rows, cols,
                        row_offset ? row_offset + qs : NULL, A, lt, b, dAt, dZ);
            for (int r = 0; r < rows; ++r) {
                N[t * block + r] = b[r];
                REAL s = 0;
                for (int c = 0; c < cols; ++c) s += dAt[r * cols + c];
                b[r] = b[r] + s;
            }
            for (int r = 0; r < rows; ++r) {
                for (int e = 0; e < d; ++e) acc[e] = 0;
                for (int c = 0; c < cols; ++c) {
                    const REAL w = dZ[r * cols + c];
                    const REAL* kc = k + (size_t)(ks + c) * d;
#pragma omp simd
                    for (int e = 0; e < d; ++e) acc[e] += w * kc[e];
                }
                REAL* dqr = dq + (size_t)(qs + r) * d;
#pragma omp simd
                for (int e = 0; e < d; ++e) dqr[e] += acc[e] * scale;
            }
        }
    }
    for (int kb = 0; kb < nb; ++kb) {
        const int ks = kb * block, ke = ks + block < L ? ks + block : L, cols = ke - ks;
        for (int qb = kb; qb < nb; ++qb) {
            if (kb < first_kb[qb]) continue; /* tile skipped by the forward */
            const int qs = qb * block, qe = qs + block < L ? qs + block : L, rows = qe - qs;
            const size_t t = (size_t)qb * (qb + 1) / 2 + kb;
            FN(sbo_tile_)(q + (size_t)qs * d, k + (size_t)ks * d, d, rows, cols, kb == qb,
                          scale, M + t * block, z, lt, A);
            FN(sbo_dz_)(d_o + (size_t)qs * d, v + (size_t)ks * d, d, rows, cols,
                        row_offset ? row_offset + qs : NULL, A, lt, N + t * block, dAt, dZ);
            /* dZ^T Q * scale and A^T dO for this tile, rows in ascending order */
            memset(tk, 0, sizeof(REAL) * (size_t)cols * d);
            memset(tv, 0, sizeof(REAL) * (size_t)cols * d);
            for (int r = 0; r < rows; ++r) {
                const REAL* qr = q + (size_t)(qs + r) * d;
                const REAL* dr = d_o + (size_t)(qs + r) * d;
                for (int c = 0; c < cols; ++c) {
                    const REAL wk = dZ[r * cols + c], wv = A[r * cols + c];
                    REAL* tkc = tk + (size_t)c * d;
                    REAL* tvc = tv + (size_t)c * d;
#pragma omp simd
                    for (int e = 0; e < d; ++e) {
                        tkc[e] += wk * qr[e];
                        tvc[e] += wv * dr[e];
                    }
                }
            }
            for (int c = 0; c < cols; ++c) {
                REAL* dkc = dk + (size_t)(ks + c) * d;
                REAL* dvc = dv + (size_t)(ks + c) * d;
#pragma omp simd
                for (int e = 0; e < d; ++e) {
                    dkc[e] += tk[(size_t)c * d + e] * scale;
                    dvc[e] += tv[(size_t)c * d + e];
                }
            }
        }
    }
    free(z); free(lt); free(A); free(dAt); free(dZ); free(b); free(acc); free(tk); free(tv);
    return 0;
}

/* Batched drivers: `units` independent (batch, head) problems, each a
 * contiguous L x d slab (no cross-head term anywhere), run
 * in parallel over host threads.  M/N are [units][n_tiles][block]. */
long long FN(sbo_forward_batch_)(int units, int L, int d, int block, const REAL* q,
                                 const REAL* k, const REAL* v, int skip, double skip_eps,
                                 REAL* o, REAL* a_out, int64_t* first_kb, REAL* M,
                                 int n_threads) {
    const int nb = (L + block - 1) / block;
    const size_t slab = (size_t)L * d, nt = (size_t)nb * (nb + 1) / 2 * block;
    long long total = 0;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total) num_threads(n_threads)
    for (int u = 0; u < units; ++u) {
        long long vis = FN(sbo_forward_)(L, d, block, q + u * slab, k + u * slab, v + u * slab,
                                         skip, skip_eps, o + u * slab, a_out + (size_t)u * L,
                                         first_kb + (size_t)u * nb, M ? M + u * nt : NULL);
        if (vis < 0) bad = 1; else total += vis;
    }
    return bad ? -1 : total;
}

int FN(sbo_backward_batch_)(int units, int L, int d, int block, const REAL* q, const REAL* k,
                            const REAL* v, const REAL* d_o, const REAL* row_offset,
                            const int64_t* first_kb, const REAL* M, REAL* N, REAL* dq,
                            REAL* dk, REAL* dv, int n_threads) {
    const int nb = (L + block - 1) / block;
    const size_t slab = (size_t)L * d, nt = (size_t)nb * (nb + 1) / 2 * block;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
    for (int u = 0; u < units; ++u) {
        int rc = FN(sbo_backward_twophase_)(
            L, d, block, q + u * slab, k + u * slab, v + u * slab, d_o + u * slab,
            row_offset ? row_offset + (size_t)u * L : NULL, first_kb + (size_t)u * nb,
            M + u * nt, N + u * nt, dq + u * slab, dk + u * slab, dv + u * slab);
        if (rc) bad = 1;
    }
    return bad ? -1 : 0;
}

#undef FN
#undef CAT
#undef CAT_
