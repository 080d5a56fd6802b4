// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers (for ctypes) around the reference LPD-SVM sources, which
// oracle/Makefile compiles unmodified from /root/reference/proj/src against the
// Eigen-subset substitute (oracle/eigen_subset). Used to pin oracle/lpd_oracle.c
// and as the "reference" CPU baseline of bench.py. Never linked into the product.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lpdsvm/dataio.hpp"
#include "lpdsvm/dcd.hpp"
#include "lpdsvm/factor.hpp"
#include "lpdsvm/kernel.hpp"
#include "lpdsvm/multiclass.hpp"
#include "lpdsvm/parallel.hpp"

using namespace lpdsvm;

namespace {
thread_local std::string g_err;

std::vector<SparseVector> from_csr(int64_t n, const int64_t* ptr, const int32_t* idx,
                                   const double* val) {
    std::vector<SparseVector> pts(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        SparseVector& p = pts[static_cast<size_t>(i)];
        p.reserve(static_cast<size_t>(ptr[i + 1] - ptr[i]));
        for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) p.push_back({idx[e], val[e]});
    }
    return pts;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

struct FactorHandle {
    LowRankFactor factor;
    FactorTimings timings;
};
}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() { return g_err.c_str(); }
__attribute__((visibility("default"))) int ref_hardware_threads() { return hardware_threads(); }

// kernel.cpp:17-19
__attribute__((visibility("default"))) double ref_gaussian(int64_t na, const int32_t* ia,
                                                           const double* va, int64_t nb,
                                                           const int32_t* ib, const double* vb,
                                                           double gamma) {
    SparseVector a, b;
    for (int64_t i = 0; i < na; ++i) a.push_back({ia[i], va[i]});
    for (int64_t i = 0; i < nb; ++i) b.push_back({ib[i], vb[i]});
    return gaussian(a, b, {KernelKind::Gaussian, gamma});
}

// kernel.cpp:21-25 + kernel.cpp:31-57 (norms computed by the reference itself)
__attribute__((visibility("default"))) int ref_kernel_block(int64_t m, const int64_t* a_ptr,
                                                            const int32_t* a_idx, const double* a_val,
                                                            int64_t nb, const int64_t* b_ptr,
                                                            const int32_t* b_idx, const double* b_val,
                                                            double gamma, int threads, double* out) {
    return guard([&] {
        auto A = from_csr(m, a_ptr, a_idx, a_val);
        auto Bv = from_csr(nb, b_ptr, b_idx, b_val);
        Matrix K = kernel_block(A, Bv, {KernelKind::Gaussian, gamma}, threads);
        std::memcpy(out, K.data(), sizeof(double) * static_cast<size_t>(m * nb));
    });
}

__attribute__((visibility("default"))) int ref_squared_norms(int64_t n, const int64_t* ptr,
                                                             const int32_t* idx, const double* val,
                                                             double* out) {
    return guard([&] {
        auto P = from_csr(n, ptr, idx, val);
        auto v = squared_norms(P);
        std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(n));
    });
}

// factor.cpp:83-110 — the hot path itself, reference implementation.
__attribute__((visibility("default"))) int ref_compute_g(
    int64_t n, const int64_t* x_ptr, const int32_t* x_idx, const double* x_val, int64_t b,
    const int64_t* l_ptr, const int32_t* l_idx, const double* l_val, const double* L,
    int64_t b_eff, double gamma, int64_t chunk_size, int threads, double* G, double* seconds) {
    return guard([&] {
        auto X = from_csr(n, x_ptr, x_idx, x_val);
        auto Y = from_csr(b, l_ptr, l_idx, l_val);
        Matrix Lm(static_cast<size_t>(b), static_cast<size_t>(b_eff));
        std::memcpy(Lm.data(), L, sizeof(double) * static_cast<size_t>(b * b_eff));
        const KernelParams params{KernelKind::Gaussian, gamma};
        validate(params);
        const auto t0 = std::chrono::steady_clock::now();
        // same sequence as build_factor_with_landmarks' gmatrix stage (factor.cpp:129-133)
        std::vector<double> ln = squared_norms(Y);
        std::vector<double> xn = squared_norms(X);
        Matrix Gm = compute_G(X, xn, Y, ln, Lm, params, static_cast<size_t>(chunk_size), threads);
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(G, Gm.data(), sizeof(double) * static_cast<size_t>(n * b_eff));
    });
}

// factor.cpp:27-31
__attribute__((visibility("default"))) int64_t ref_select_landmarks(int64_t n, int64_t budget,
                                                                    uint64_t seed, int32_t* out) {
    int64_t k = -1;
    guard([&] {
        auto ids = select_landmarks(static_cast<size_t>(n), static_cast<size_t>(budget), seed);
        for (size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
        k = static_cast<int64_t>(ids.size());
    });
    return k;
}

// factor.cpp:112-143 with caller-fixed landmarks; returns an opaque handle.
__attribute__((visibility("default"))) void* ref_factor_with_landmarks(
    int64_t n, const int64_t* x_ptr, const int32_t* x_idx, const double* x_val, int64_t b,
    const int64_t* l_ptr, const int32_t* l_idx, const double* l_val, double gamma, double tau,
    int64_t chunk_size, int threads, int64_t* b_eff, double* prep_seconds, double* gmat_seconds) {
    FactorHandle* h = nullptr;
    const int rc = guard([&] {
        auto X = from_csr(n, x_ptr, x_idx, x_val);
        auto Y = from_csr(b, l_ptr, l_idx, l_val);
        FactorOptions opt;
        opt.tau_rel = tau;
        opt.chunk_size = static_cast<size_t>(chunk_size);
        opt.num_threads = threads;
        auto* hh = new FactorHandle();
        try {
            hh->factor = build_factor_with_landmarks(X, std::move(Y), {}, {KernelKind::Gaussian, gamma},
                                                     opt, &hh->timings);
        } catch (...) {
            delete hh;
            throw;
        }
        h = hh;
    });
    if (rc != 0) return nullptr;
    *b_eff = h->factor.b_eff;
    if (prep_seconds) *prep_seconds = h->timings.preparation_seconds;
    if (gmat_seconds) *gmat_seconds = h->timings.gmatrix_seconds;
    return h;
}

// factor.cpp:145-153 (landmarks sampled by the reference)
__attribute__((visibility("default"))) void* ref_build_factor(
    int64_t n, const int64_t* x_ptr, const int32_t* x_idx, const double* x_val, int64_t budget,
    double gamma, double tau, int64_t chunk_size, int threads, uint64_t seed, int64_t* b_eff,
    int64_t* num_landmarks, double* prep_seconds, double* gmat_seconds) {
    FactorHandle* h = nullptr;
    const int rc = guard([&] {
        Dataset data;
        data.points = from_csr(n, x_ptr, x_idx, x_val);
        data.labels.assign(static_cast<size_t>(n), 1.0);
        FactorOptions opt;
        opt.budget = static_cast<size_t>(budget);
        opt.tau_rel = tau;
        opt.chunk_size = static_cast<size_t>(chunk_size);
        opt.num_threads = threads;
        opt.seed = seed;
        auto* hh = new FactorHandle();
        try {
            hh->factor = build_factor(data, {KernelKind::Gaussian, gamma}, opt, &hh->timings);
        } catch (...) {
            delete hh;
            throw;
        }
        h = hh;
    });
    if (rc != 0) return nullptr;
    *b_eff = h->factor.b_eff;
    *num_landmarks = static_cast<int64_t>(h->factor.landmarks.size());
    if (prep_seconds) *prep_seconds = h->timings.preparation_seconds;
    if (gmat_seconds) *gmat_seconds = h->timings.gmatrix_seconds;
    return h;
}

// Copies L (B x b_eff), G (n x b_eff) and landmark ids (may be empty) out of a handle.
__attribute__((visibility("default"))) void ref_factor_copy(void* hp, double* L, double* G,
                                                            int32_t* ids) {
    auto* h = static_cast<FactorHandle*>(hp);
    if (L) std::memcpy(L, h->factor.L.data(), sizeof(double) * h->factor.L.rows() * h->factor.L.cols());
    if (G) std::memcpy(G, h->factor.G.data(), sizeof(double) * h->factor.G.rows() * h->factor.G.cols());
    if (ids)
        for (size_t i = 0; i < h->factor.landmark_ids.size(); ++i) ids[i] = h->factor.landmark_ids[i];
}

__attribute__((visibility("default"))) void ref_factor_free(void* hp) {
    delete static_cast<FactorHandle*>(hp);
}

// multiclass.cpp:153-168
__attribute__((visibility("default"))) int ref_vote(const double* decisions, int64_t num_pairs,
                                                    int64_t num_classes) {
    return vote(std::span<const double>(decisions, static_cast<size_t>(num_pairs)),
                static_cast<size_t>(num_classes));
}

// dcd.cpp:60-89 (make_binary_problem) + dcd.cpp:212-259 (solve_binary) over every row of
// a caller-given G (n x b_eff, row-major): the reference's stage-2 solver, unchanged, so
// the downstream effect of a G from another implementation can be measured with the
// solver held fixed. report6 = {dual_objective, epochs, coordinate_visits,
// final_violation, converged, shrunk_peak}.
__attribute__((visibility("default"))) int ref_solve_binary(
    int64_t n, int64_t b_eff, const double* G, const double* y, double C, double eps,
    int64_t max_epochs, int shrinking, uint64_t seed, uint64_t problem_tag,
    const double* warm_alpha, double* alpha_out, double* w_out, double* report6) {
    return guard([&] {
        Matrix Gm(static_cast<size_t>(n), static_cast<size_t>(b_eff));
        std::memcpy(Gm.data(), G, sizeof(double) * static_cast<size_t>(n * b_eff));
        std::vector<int> rows(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) rows[static_cast<size_t>(i)] = static_cast<int>(i);
        BinaryProblem problem =
            make_binary_problem(Gm, std::move(rows), std::vector<double>(y, y + n), C);
        SolveOptions opt;
        opt.eps = eps;
        opt.max_epochs = max_epochs;
        opt.shrinking = shrinking != 0;
        opt.seed = seed;
        opt.problem_tag = problem_tag;
        std::span<const double> warm;
        if (warm_alpha) warm = std::span<const double>(warm_alpha, static_cast<size_t>(n));
        SolveResult r = solve_binary(problem, Gm, opt, warm);
        std::memcpy(alpha_out, r.alpha.data(), sizeof(double) * r.alpha.size());
        std::memcpy(w_out, r.w.data(), sizeof(double) * r.w.size());
        report6[0] = r.report.dual_objective;
        report6[1] = static_cast<double>(r.report.epochs);
        report6[2] = static_cast<double>(r.report.coordinate_visits);
        report6[3] = r.report.final_violation;
        report6[4] = r.report.converged ? 1.0 : 0.0;
        report6[5] = static_cast<double>(r.report.shrunk_peak);
    });
}

}  // extern "C"
