// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libhexfuse_ref.so.  Used (1) to pin the C restatement
// oracle/hexfuse_oracle.c bit-for-bit, (2) to generate tests/golden/, and
// (3) as the CPU baseline ("kind": "reference") in bench.py.  The shipped
// B200 library never links it.
//
// Every function wraps exactly one reference entry point:
//   ref_random_field       -> hexfuse::random_field        (oracle.hpp:154-166)
//   ref_tgv_field          -> hexfuse::tgv_field           (oracle.hpp:116-151)
//   ref_oracle_divergence  -> hexfuse::oracle_divergence   (oracle.hpp:20-62)
//   ref_field_rel_error    -> hexfuse::field_rel_error     (verify.hpp:19-33)
//   ref_gl_derivative      -> gauss_legendre_points + derivative_matrix (operators.hpp:17-74)
//   ref_derivative_matrix  -> derivative_matrix on caller nodes (operators.hpp:49-74): pins the
//                             m = 9 operator of d2 p8, whose nodes the reference does not generate
//   ref_time_oracle_mt     -> oracle_divergence on T group-aligned sub-fields, one
//                             std::thread each (the function is pure)
//   ref_export_blob        -> hexfuse::export_blob        (layout.hpp:161-177)
//   ref_import_blob        -> hexfuse::import_blob        (layout.hpp:179-200): shape into
//                             shape[5] = {d, p, n_elem, group, fp32}, words into `out`
//   ref_max_abs_eigenvalue -> max |eigenvalues(flux_jacobian(s, params, e_a))|
//                             (equations.hpp:112-130, eig.hpp:15): pins the Rusanov
//                             wave speed of the FR interface stage (hexfuse_oracle.c)
#include <hexfuse/oracle.hpp>
#include <hexfuse/verify.hpp>
#include <hexfuse/eig.hpp>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

using namespace hexfuse;

namespace {

thread_local std::string g_err;

// A StateField whose AoSoA group is exactly `group` (StateField ctor, layout.hpp:111-116).
StateField make_field(int d, int p, int n_elem, int group, int fp32) {
    return StateField(d, p, n_elem, group, fp32 ? Precision::fp32 : Precision::fp64);
}

// An ElementConfig whose elems_per_block() == group (lines: block = n*(p+1)^2, layout.hpp:76-81).
ElementConfig make_cfg(int d, int p, int n_elem, int group, int fp32) {
    ElementConfig cfg;
    cfg.d = d;
    cfg.p = p;
    cfg.n_elem = n_elem;
    cfg.method = Method::Lines;
    cfg.block_threads = group * (p + 1) * (p + 1);
    cfg.precision = fp32 ? Precision::fp32 : Precision::fp64;
    return cfg;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_random_field(int d, int p, int n_elem, int group, int fp32, unsigned long long seed, double* out) {
    return guarded([&] {
        const StateField f = random_field(make_cfg(d, p, n_elem, group, fp32), seed);
        std::memcpy(out, f.data.data(), f.data.size() * sizeof(double));
    });
}

int ref_tgv_field(int p, int n_elem, int group, int fp32, double width, int zero_mean_pressure, double* out) {
    return guarded([&] {
        TgvGrid grid;
        grid.elems = factor3(n_elem);
        grid.width = {width, width, width};
        const StateField f = tgv_field(make_cfg(3, p, n_elem, group, fp32), grid, 1.4, 0.08, zero_mean_pressure != 0);
        std::memcpy(out, f.data.data(), f.data.size() * sizeof(double));
    });
}

void ref_factor3(int n, int* out3) {
    const auto f = factor3(n);
    out3[0] = f[0];
    out3[1] = f[1];
    out3[2] = f[2];
}

int ref_oracle_divergence(int d, int p, int n_elem, int group, int fp32, const double* U, double* out, double nu,
                          double zeta, double T, const double* jac, int with_source) {
    return guarded([&] {
        StateField f = make_field(d, p, n_elem, group, fp32);
        std::memcpy(f.data.data(), U, f.data.size() * sizeof(double));
        const StateField r = oracle_divergence(f, PhysParams{nu, zeta, T}, {jac[0], jac[1], jac[2]}, with_source != 0);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(double));
    });
}

double ref_field_rel_error(int d, int p, int n_elem, int group, const double* got, const double* ref) {
    StateField a = make_field(d, p, n_elem, group, 0), b = make_field(d, p, n_elem, group, 0);
    std::memcpy(a.data.data(), got, a.data.size() * sizeof(double));
    std::memcpy(b.data.data(), ref, b.data.size() * sizeof(double));
    return field_rel_error(a, b);
}

int ref_gl_derivative(int m, double* nodes, double* D) {
    return guarded([&] {
        const auto x = gauss_legendre_points(m);
        const Matrix M = derivative_matrix(x);
        std::copy(x.begin(), x.end(), nodes);
        std::copy(M.a.begin(), M.a.end(), D);
    });
}

int ref_derivative_matrix(int m, const double* nodes, double* D) {
    return guarded([&] {
        const Matrix M = derivative_matrix(std::vector<double>(nodes, nodes + m));
        std::copy(M.a.begin(), M.a.end(), D);
    });
}

// Time the reference oracle over `n_threads` contiguous, group-aligned element
// ranges of U.  Sub-field construction (data copies) is outside the timed
// region; only the oracle_divergence calls are timed.  Writes the assembled
// result into `out` (same layout as U) and returns wall seconds, < 0 on error.
double ref_time_oracle_mt(int d, int p, int n_elem, int group, int fp32, const double* U, double* out, double nu,
                          double zeta, double T, const double* jac, int with_source, int n_threads) {
    try {
        const StateField whole = make_field(d, p, n_elem, group, fp32);
        const int n_groups = whole.n_groups();
        const std::int64_t gw = whole.group_words();
        n_threads = std::max(1, std::min(n_threads, n_groups));
        std::vector<StateField> parts;
        std::vector<int> g0(static_cast<std::size_t>(n_threads) + 1);
        for (int t = 0; t <= n_threads; ++t) g0[static_cast<std::size_t>(t)] = static_cast<int>(
            static_cast<std::int64_t>(n_groups) * t / n_threads);
        for (int t = 0; t < n_threads; ++t) {
            const int ga = g0[static_cast<std::size_t>(t)], gb = g0[static_cast<std::size_t>(t) + 1];
            const int e0 = ga * group, e1 = std::min(n_elem, gb * group);
            StateField f = make_field(d, p, e1 - e0, group, fp32);
            std::memcpy(f.data.data(), U + static_cast<std::int64_t>(ga) * gw, f.data.size() * sizeof(double));
            parts.push_back(std::move(f));
        }
        std::vector<StateField> results(parts.size());
        const PhysParams par{nu, zeta, T};
        const std::array<double, 3> j3{jac[0], jac[1], jac[2]};
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < n_threads; ++t)
            pool.emplace_back([&, t] {
                results[static_cast<std::size_t>(t)] =
                    oracle_divergence(parts[static_cast<std::size_t>(t)], par, j3, with_source != 0);
            });
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        for (int t = 0; t < n_threads; ++t) {
            const auto& r = results[static_cast<std::size_t>(t)];
            std::memcpy(out + static_cast<std::int64_t>(g0[static_cast<std::size_t>(t)]) * gw, r.data.data(),
                        r.data.size() * sizeof(double));
        }
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

int ref_export_blob(int d, int p, int n_elem, int group, int fp32, const double* data, const char* path) {
    return guarded([&] {
        StateField f = make_field(d, p, n_elem, group, fp32);
        std::memcpy(f.data.data(), data, f.data.size() * sizeof(double));
        export_blob(f, path);
    });
}

// shape[5] = {d, p, n_elem, group, fp32}; `out` (may be null: shape only) receives
// min(capacity, words) doubles.  Returns the field's word count, < 0 on error.
long long ref_import_blob(const char* path, int* shape, double* out, long long capacity) {
    long long words = -1;
    const int rc = guarded([&] {
        const StateField f = import_blob(path);
        shape[0] = f.d;
        shape[1] = f.p;
        shape[2] = f.n_elem;
        shape[3] = f.group;
        shape[4] = f.precision == Precision::fp32 ? 1 : 0;
        words = static_cast<long long>(f.data.size());
        if (out) std::memcpy(out, f.data.data(), static_cast<std::size_t>(std::min(words, capacity)) * sizeof(double));
    });
    return rc == 0 ? words : -rc;
}

double ref_max_abs_eigenvalue(int d, const double* s, int a, double nu, double zeta, double T) {
    double r = -1.0;
    guarded([&] {
        AcmHdState st(d);
        for (int v = 0; v < n_vars(d); ++v) st.v[static_cast<std::size_t>(v)] = s[v];
        PhysParams par{nu, zeta, T};
        std::vector<double> dir(static_cast<std::size_t>(d), 0.0);
        dir[static_cast<std::size_t>(a)] = 1.0;
        r = 0.0;
        for (const auto& ev : eigenvalues(flux_jacobian(st, par, dir))) r = std::max(r, std::abs(ev));
    });
    return r;
}

}  // extern "C"
