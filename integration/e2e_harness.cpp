// e2e_harness.cpp — what a C++ user of the reference library does, timed. Compiled twice
// from this one source (integration/Makefile, oracle/Makefile):
//
//   integration/_build/libe2e_b200.so  against the drop-in build (reference objects with
//                                      compute_G & co. served by liblpd_nystrom.so)
//   oracle/_ref/libe2e_ref.so          against the reference objects, unmodified
//
// so bench.py measures the reference's own public C++ API — build_factor / compute_G /
// ovo_train / ovo_predict (factor.hpp:50-80, multiclass.hpp:70-82) — on both builds with
// the same inputs and the same host code around it. Inputs arrive as CSR (the flattened
// std::vector<Feature>, dataio.hpp:14-24) and are turned into SparseVectors outside the
// timed regions, as a caller's data would already be.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lpdsvm/dataio.hpp"
#include "lpdsvm/factor.hpp"
#include "lpdsvm/kernel.hpp"
#include "lpdsvm/multiclass.hpp"
#include "lpdsvm/parallel.hpp"

using namespace lpdsvm;

namespace {
thread_local std::string g_err;
using clk = std::chrono::steady_clock;
double since(clk::time_point t) { return std::chrono::duration<double>(clk::now() - t).count(); }

std::vector<SparseVector> rows_from_csr(int64_t n, const int64_t* ptr, const int32_t* idx, const double* val) {
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
}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* e2e_last_error() { return g_err.c_str(); }
__attribute__((visibility("default"))) int e2e_hardware_threads() { return hardware_threads(); }

// The gmatrix stage of build_factor_with_landmarks (factor.cpp:129-133): squared_norms of
// the points, then compute_G into a fresh Matrix, exactly as the reference calls it.
// seconds[0] = the stage (norms + compute_G), seconds[1] = compute_G alone,
// seconds[2] = destroying the returned Matrix (not part of the stage).
// The first `sample_rows` rows of G are copied to sample (may be NULL).
__attribute__((visibility("default"))) int e2e_compute_g(
    int64_t n, const int64_t* xp, const int32_t* xi, const double* xv, int64_t b, const int64_t* lp,
    const int32_t* li, const double* lv, const double* L, int64_t b_eff, double gamma, int64_t chunk,
    int threads, int64_t sample_rows, double* sample, double* seconds) {
    return guard([&] {
        std::vector<SparseVector> points = rows_from_csr(n, xp, xi, xv);
        std::vector<SparseVector> landmarks = rows_from_csr(b, lp, li, lv);
        Matrix Lm(static_cast<size_t>(b), static_cast<size_t>(b_eff));
        std::memcpy(Lm.data(), L, sizeof(double) * static_cast<size_t>(b * b_eff));
        const KernelParams params{KernelKind::Gaussian, gamma};
        std::vector<double> landmark_norms = squared_norms(landmarks);  // preparation stage
        const auto t0 = clk::now();
        std::vector<double> norms = squared_norms(points);
        const auto t1 = clk::now();
        Matrix G = compute_G(points, norms, landmarks, landmark_norms, Lm, params,
                             static_cast<size_t>(chunk), threads);
        seconds[0] = since(t0);
        seconds[1] = since(t1);
        if (sample && sample_rows > 0)
            std::memcpy(sample, G.data(), sizeof(double) * static_cast<size_t>(sample_rows * b_eff));
        const auto t2 = clk::now();
        { Matrix drop = std::move(G); }
        seconds[2] = since(t2);
    });
}

// train_impl (bindings/module.cpp:35-78) for the Python `lpdsvm.train`, then
// Model.error_rate on a test set (module.cpp:144-156 → ovo_predict). out[]:
//   0 train wall seconds (build_factor + ovo_train, as lpdsvm.train times them)
//   1 preparation_seconds  2 gmatrix_seconds  3 training_seconds (module.cpp:64-69)
//   4 predict seconds      5 test error rate  6 epochs  7 b_eff
//   8 unconverged pairs    9 dual objective of pair 0  10 coordinate visits
__attribute__((visibility("default"))) int e2e_train(
    int64_t n, const int64_t* xp, const int32_t* xi, const double* xv, const double* labels,
    int64_t n_test, const int64_t* tp, const int32_t* ti, const double* tv, const double* test_labels,
    int64_t budget, double C, double gamma, double eps, double tau, int threads, uint64_t seed, double* out) {
    return guard([&] {
        Dataset data;
        data.points = rows_from_csr(n, xp, xi, xv);
        data.labels.assign(labels, labels + n);
        std::vector<SparseVector> test = rows_from_csr(n_test, tp, ti, tv);
        if (threads < 1) threads = hardware_threads();

        const auto t0 = clk::now();
        LabelMap label_map = build_label_map(data.labels);
        FactorOptions fo;
        fo.budget = static_cast<size_t>(budget);
        fo.tau_rel = tau;
        fo.num_threads = threads;
        fo.seed = seed;
        FactorTimings timings;
        LowRankFactor factor = build_factor(data, {KernelKind::Gaussian, gamma}, fo, &timings);
        OvoTrainOptions to;
        to.solve.eps = eps;
        to.solve.seed = seed;
        to.num_threads = threads;
        const auto t1 = clk::now();
        OvoTrainResult trained = ovo_train(factor, data.labels, label_map, C, to);
        out[3] = since(t1);
        out[0] = since(t0);
        out[1] = timings.preparation_seconds;
        out[2] = timings.gmatrix_seconds;

        const auto t2 = clk::now();
        std::vector<double> pred = ovo_predict(trained.model, test, threads);
        out[4] = since(t2);
        int64_t wrong = 0;
        for (int64_t i = 0; i < n_test; ++i)
            if (pred[static_cast<size_t>(i)] != test_labels[i]) ++wrong;
        out[5] = n_test > 0 ? static_cast<double>(wrong) / static_cast<double>(n_test) : 0.0;
        long long epochs = 0, visits = 0, unconverged = 0;
        for (const SolveReport& r : trained.reports) {
            epochs += r.epochs;
            visits += r.coordinate_visits;
            if (!r.converged) ++unconverged;
        }
        out[6] = static_cast<double>(epochs);
        out[7] = static_cast<double>(factor.b_eff);
        out[8] = static_cast<double>(unconverged);
        out[9] = trained.reports.empty() ? 0.0 : trained.reports[0].dual_objective;
        out[10] = static_cast<double>(visits);
    });
}

}  // extern "C"
