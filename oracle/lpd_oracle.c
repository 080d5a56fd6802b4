/*
 * lpd_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C, fp64 restatement of the reference LPD-SVM factor path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg to check the
 * B200 library. Nothing in paper_2207_01016_b200/ links or calls this file.
 *
 * Each function cites the reference code it restates (paths relative to
 * /root/reference/proj). Pinning: tests/test_oracle.py checks these functions
 * against the SPEC.md known answers and against the reference's own sources
 * compiled unmodified (oracle/_ref, built by oracle/Makefile), bit-exact for
 * kernel_block / squared norms and to <= 1e-12 relative for compute_G (the
 * reference GEMM is Eigen's, whose summation order is not specified).
 *
 * Sparse points use CSR (indptr int64[n+1], indices int32 0-based strictly
 * ascending per row, values fp64), the flattened reference SparseVector
 * (include/lpdsvm/dataio.hpp:14-24).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_API __attribute__((visibility("default")))

/* dataio.cpp:15-30 — sparse merge-join inner product. */
static double sp_dot(const int32_t* ia, const double* va, int64_t na, const int32_t* ib,
                     const double* vb, int64_t nb) {
    double r = 0.0;
    int64_t i = 0, j = 0;
    while (i < na && j < nb) {
        if (ia[i] == ib[j]) {
            r += va[i] * vb[j];
            ++i;
            ++j;
        } else if (ia[i] < ib[j]) {
            ++i;
        } else {
            ++j;
        }
    }
    return r;
}

/* dataio.cpp:32-36 */
static double sp_squared_norm(const double* v, int64_t n) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += v[i] * v[i];
    return r;
}

/* dataio.cpp:38-58 — direct squared distance (used by gaussian(), kernel.cpp:17-19). */
static double sp_squared_distance(const int32_t* ia, const double* va, int64_t na,
                                  const int32_t* ib, const double* vb, int64_t nb) {
    double r = 0.0;
    int64_t i = 0, j = 0;
    while (i < na && j < nb) {
        if (ia[i] == ib[j]) {
            double d = va[i] - vb[j];
            r += d * d;
            ++i;
            ++j;
        } else if (ia[i] < ib[j]) {
            r += va[i] * va[i];
            ++i;
        } else {
            r += vb[j] * vb[j];
            ++j;
        }
    }
    for (; i < na; ++i) r += va[i] * va[i];
    for (; j < nb; ++j) r += vb[j] * vb[j];
    return r;
}

/* kernel.cpp:21-25 — squared_norms over CSR rows. */
ORA_API void ora_squared_norms(int64_t n, const int64_t* indptr, const double* values,
                               double* out) {
    for (int64_t i = 0; i < n; ++i)
        out[i] = sp_squared_norm(values + indptr[i], indptr[i + 1] - indptr[i]);
}

/* kernel.cpp:17-19 — gaussian(a, b) = exp(-gamma * squared_distance(a, b)). */
ORA_API double ora_gaussian(const int32_t* ia, const double* va, int64_t na, const int32_t* ib,
                            const double* vb, int64_t nb, double gamma) {
    return exp(-gamma * sp_squared_distance(ia, va, na, ib, vb, nb));
}

/* kernel.cpp:31-57 — kernel_block via the norm expansion, clamp at 0 (:49-51), exp.
 * out is m x nb row-major. */
ORA_API void ora_kernel_block(int64_t m, const int64_t* a_ptr, const int32_t* a_idx,
                              const double* a_val, const double* norms_a, int64_t nb,
                              const int64_t* b_ptr, const int32_t* b_idx, const double* b_val,
                              const double* norms_b, double gamma, double* out) {
    for (int64_t i = 0; i < m; ++i) {
        const int32_t* ia = a_idx + a_ptr[i];
        const double* va = a_val + a_ptr[i];
        const int64_t na = a_ptr[i + 1] - a_ptr[i];
        double* o = out + i * nb;
        for (int64_t j = 0; j < nb; ++j) {
            double d2 = norms_a[i] + norms_b[j] -
                        2.0 * sp_dot(ia, va, na, b_idx + b_ptr[j], b_val + b_ptr[j],
                                     b_ptr[j + 1] - b_ptr[j]);
            if (d2 < 0.0) d2 = 0.0;
            o[j] = exp(-gamma * d2);
        }
    }
}

/* factor.cpp:83-110 — compute_G: per chunk of chunk_size rows, Z = kernel_block(chunk,
 * landmarks) then G[chunk] = Z * L (fp64). L is b x b_eff row-major; G is n x b_eff
 * row-major. The GEMM sums over landmarks in ascending order. Returns 0, or -1 on the
 * reference's std::invalid_argument conditions (factor.cpp:87, 173 is the caller's
 * shape check) or -2 on allocation failure. */
ORA_API int ora_compute_g(int64_t n, const int64_t* x_ptr, const int32_t* x_idx,
                          const double* x_val, const double* norms, int64_t b,
                          const int64_t* l_ptr, const int32_t* l_idx, const double* l_val,
                          const double* l_norms, const double* L, int64_t b_eff, double gamma,
                          int64_t chunk_size, double* G) {
    if (chunk_size <= 0) return -1;
    if (!(gamma > 0.0) || !isfinite(gamma)) return -1;
    double* Z = (double*)malloc(sizeof(double) * (size_t)(chunk_size < n ? chunk_size : (n > 0 ? n : 1)) * (size_t)(b > 0 ? b : 1));
    if (!Z) return -2;
    for (int64_t begin = 0; begin < n; begin += chunk_size) {
        const int64_t rows = (n - begin) < chunk_size ? (n - begin) : chunk_size;
        ora_kernel_block(rows, x_ptr + begin, x_idx, x_val, norms + begin, b, l_ptr, l_idx, l_val,
                         l_norms, gamma, Z);
        for (int64_t i = 0; i < rows; ++i) {
            double* g = G + (begin + i) * b_eff;
            for (int64_t k = 0; k < b_eff; ++k) g[k] = 0.0;
            const double* z = Z + i * b;
            for (int64_t j = 0; j < b; ++j) {
                const double zj = z[j];
                const double* lrow = L + j * b_eff;
                for (int64_t k = 0; k < b_eff; ++k) g[k] += zj * lrow[k];
            }
        }
    }
    free(Z);
    return 0;
}

/* modelsel.cpp:123-140 — held-out scoring d[r][p] = G_r . w_p, fp64, j ascending.
 * G rows selected by row_ids (n_rows of them); W is P x b_eff; D is n_rows x P. */
ORA_API void ora_decision_values(int64_t n_rows, const int64_t* row_ids, const double* G,
                                 int64_t ldg, int64_t b_eff, const double* W, int64_t P,
                                 double* D) {
    for (int64_t r = 0; r < n_rows; ++r) {
        const double* g = G + (row_ids ? row_ids[r] : r) * ldg;
        for (int64_t p = 0; p < P; ++p) {
            const double* w = W + p * b_eff;
            double d = 0.0;
            for (int64_t j = 0; j < b_eff; ++j) d += g[j] * w[j];
            D[r * P + p] = d;
        }
    }
}

/* multiclass.cpp:153-168 — one-vs-one vote: strictly positive votes for class a,
 * otherwise class b; ties to the smaller class index. */
ORA_API int ora_vote(const double* decisions, int64_t num_classes) {
    int votes_stack[64];
    int* votes = num_classes <= 64 ? votes_stack : (int*)calloc((size_t)num_classes, sizeof(int));
    if (!votes) return -1;
    memset(votes, 0, sizeof(int) * (size_t)num_classes);
    int64_t p = 0;
    for (int64_t a = 0; a < num_classes; ++a)
        for (int64_t b = a + 1; b < num_classes; ++b, ++p) {
            if (decisions[p] > 0.0)
                ++votes[a];
            else
                ++votes[b];
        }
    int best = 0;
    for (int64_t c = 1; c < num_classes; ++c)
        if (votes[c] > votes[best]) best = (int)c;
    if (votes != votes_stack) free(votes);
    return best;
}

/* rng.hpp:11-25 — splitmix64 finaliser and combine_seed. */
static uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
ORA_API uint64_t ora_combine_seed(uint64_t seed, uint64_t tag) {
    return mix64(seed ^ (mix64(tag) + 0x9e3779b97f4a7c15ULL + (seed << 6) + (seed >> 2)));
}

/* std::mt19937_64 (the engine rng.hpp:30-57 wraps; its output sequence is fixed by
 * the C++ standard, [rand.predef]). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;
static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}
static uint64_t mt64_next(mt64* s) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}
/* rng.hpp:36-45 — unbiased draw from [0, n). */
static uint64_t rng_below(mt64* s, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t r;
    do {
        r = mt64_next(s);
    } while (r >= limit);
    return r % n;
}

/* factor.cpp:27-31 + rng.hpp:60-72 — select_landmarks(n, budget, seed):
 * first min(budget, n) entries of a seeded partial Fisher-Yates permutation,
 * seed tag 0x1a2d. Returns the count written (or -1 on invalid input). */
ORA_API int64_t ora_select_landmarks(int64_t n, int64_t budget, uint64_t seed, int32_t* out) {
    if (budget <= 0 || n <= 0) return -1;
    int32_t* pool = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    if (!pool) return -1;
    for (int64_t i = 0; i < n; ++i) pool[i] = (int32_t)i;
    mt64 s;
    mt64_seed(&s, ora_combine_seed(seed, 0x1a2dULL));
    const int64_t k = budget > n ? n : budget;
    for (int64_t i = 0; i < k; ++i) {
        const int64_t j = i + (int64_t)rng_below(&s, (uint64_t)(n - i));
        int32_t t = pool[i];
        pool[i] = pool[j];
        pool[j] = t;
    }
    memcpy(out, pool, sizeof(int32_t) * (size_t)k);
    free(pool);
    return k;
}
