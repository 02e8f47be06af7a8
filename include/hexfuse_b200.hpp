// hexfuse_b200.hpp -- header-only C++ adapter that makes the B200 kernels a
// drop-in for the reference's host entry point
//
//     StateField hexfuse::oracle_divergence(const StateField& U, const PhysParams& params,
//                                           const std::array<double, 3>& jac, bool with_source);
//     (/root/reference/proj/include/hexfuse/oracle.hpp:20-21)
//
// as
//
//     StateField hexfuse_b200::fused_divergence_b200(U, params, jac, with_source [, method]);
//
// It is templated on the caller's StateField / PhysParams types so it binds to
// the reference's own structs (layout.hpp:104-153, equations.hpp:14-24) without
// this repository including -- or copying -- any reference header.  Required
// members, exactly the reference's: U.d, U.p, U.n_elem, U.group, U.precision
// (enum whose first enumerator is fp32, core.hpp:10), U.data (std::vector<double>);
// params.nu, params.zeta, params.T, params.validate().
//
// Semantics match the reference: the result is a copy of U's shape and group,
// zeroed, then filled (oracle.hpp:26-27); FP32 fields cross the ABI as float,
// converted exactly as export_blob does (layout.hpp:166-170); invalid input
// throws std::invalid_argument, device failures throw std::runtime_error.
#pragma once

#include <algorithm>
#include <array>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hexfuse_b200.h"

namespace hexfuse_b200 {

namespace detail {

struct ContextDeleter {
    void operator()(hf_context* c) const { hf_context_destroy(c); }
};

// One host-path context per thread (device 0 unless set_device() was called).
inline int& thread_device() {
    thread_local int dev = 0;
    return dev;
}

inline hf_context* thread_context() {
    thread_local std::unique_ptr<hf_context, ContextDeleter> ctx;
    thread_local int ctx_dev = -1;
    if (!ctx || ctx_dev != thread_device()) {
        ctx.reset(hf_context_create(thread_device()));
        ctx_dev = thread_device();
        if (!ctx) throw std::runtime_error(std::string("hf_context_create: ") + hf_last_error());
    }
    return ctx.get();
}

inline void check(int rc, const char* what) {
    if (rc == HF_OK) return;
    const std::string msg = std::string(what) + ": " + hf_last_error();
    if (rc == HF_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

}  // namespace detail

inline void set_device(int device) { detail::thread_device() = device; }

// The reference's kernel method (layout.hpp:18, enum class Method { PlanarUnmanaged,
// PlanarManaged, Lines }) -> HF_METHOD_*.  Templated on the caller's enum so that this
// header does not include the reference's.
template <class MethodEnum>
int method_of(MethodEnum m) {
    switch (static_cast<int>(m)) {
        case 0: return HF_METHOD_PLANAR;
        case 1: return HF_METHOD_PLANAR_MANAGED;
        case 2: return HF_METHOD_LINES;
        default: throw std::invalid_argument("method_of: unknown hexfuse::Method");
    }
}

template <class StateField, class PhysParams>
hf_problem make_problem(const StateField& U, const PhysParams& params, const std::array<double, 3>& jac,
                        bool with_source, int method = HF_METHOD_AUTO) {
    hf_problem pr{};
    pr.d = U.d;
    pr.p = U.p;
    pr.n_elem = U.n_elem;
    pr.group = U.group;
    pr.precision = static_cast<int>(U.precision) == 0 ? HF_FP32 : HF_FP64;  // Precision{fp32, fp64}
    pr.nu = params.nu;
    pr.zeta = params.zeta;
    pr.T = params.T;
    pr.jac[0] = jac[0];
    pr.jac[1] = jac[1];
    pr.jac[2] = jac[2];
    pr.with_source = with_source ? 1 : 0;
    pr.method = method;
    return pr;
}

// Drop-in for hexfuse::oracle_divergence (oracle.hpp:20-62) on the B200.
template <class StateField, class PhysParams>
StateField fused_divergence_b200(const StateField& U, const PhysParams& params, const std::array<double, 3>& jac,
                                 bool with_source, int method = HF_METHOD_AUTO) {
    params.validate();
    const hf_problem pr = make_problem(U, params, jac, with_source, method);
    detail::check(hf_validate(&pr), "fused_divergence_b200");
    StateField out = U;
    std::fill(out.data.begin(), out.data.end(), 0.0);
    if (U.n_elem == 0) return out;
    if (static_cast<int64_t>(U.data.size()) != hf_field_words(&pr))
        throw std::invalid_argument("fused_divergence_b200: field storage does not match its shape");
    hf_context* ctx = detail::thread_context();
    if (pr.precision == HF_FP32) {
        std::vector<float> in(U.data.size()), res(U.data.size());
        std::transform(U.data.begin(), U.data.end(), in.begin(), [](double x) { return static_cast<float>(x); });
        detail::check(hf_fused_divergence_host(ctx, &pr, in.data(), res.data()), "fused_divergence_b200");
        std::transform(res.begin(), res.end(), out.data.begin(), [](float x) { return static_cast<double>(x); });
    } else {
        detail::check(hf_fused_divergence_host(ctx, &pr, U.data.data(), out.data.data()), "fused_divergence_b200");
    }
    return out;
}

// ---- state blobs (layout.hpp:155-200) through the library's C ABI ----
// import_blob / export_blob with the reference's on-disk format (flat little-endian words +
// <path>.json sidecar), byte-identical to the reference's; errors as the reference's.
template <class StateField>
StateField import_blob_b200(const std::string& path) {
    hf_problem pr{};
    detail::check(hf_blob_info(path.c_str(), &pr), "import_blob");
    StateField f;
    f.d = pr.d;
    f.p = pr.p;
    f.n_elem = static_cast<int>(pr.n_elem);
    f.group = pr.group;
    f.precision = static_cast<decltype(f.precision)>(pr.precision == HF_FP32 ? 0 : 1);
    const int64_t words = hf_field_words(&pr);
    f.data.assign(static_cast<std::size_t>(words), 0.0);
    if (pr.precision == HF_FP32) {
        std::vector<float> tmp(f.data.size());
        detail::check(hf_blob_read(path.c_str(), &pr, tmp.data()), "import_blob");
        std::transform(tmp.begin(), tmp.end(), f.data.begin(), [](float x) { return static_cast<double>(x); });
    } else {
        detail::check(hf_blob_read(path.c_str(), &pr, f.data.data()), "import_blob");
    }
    return f;
}

template <class StateField>
void export_blob_b200(const StateField& f, const std::string& path) {
    hf_problem pr{};
    pr.d = f.d;
    pr.p = f.p;
    pr.n_elem = f.n_elem;
    pr.group = f.group;
    pr.precision = static_cast<int>(f.precision) == 0 ? HF_FP32 : HF_FP64;
    pr.zeta = pr.T = 1.0;  // shape only; physics is not part of the blob
    if (pr.precision == HF_FP32) {
        std::vector<float> tmp(f.data.size());
        std::transform(f.data.begin(), f.data.end(), tmp.begin(), [](double x) { return static_cast<float>(x); });
        detail::check(hf_blob_write(path.c_str(), &pr, tmp.data()), "export_blob");
    } else {
        detail::check(hf_blob_write(path.c_str(), &pr, f.data.data()), "export_blob");
    }
}

// A blob in, the divergence blob out, on the B200 (shape from the input's sidecar).
template <class PhysParams>
void fused_divergence_blob(const std::string& in_path, const std::string& out_path, const PhysParams& params,
                           const std::array<double, 3>& jac, bool with_source, int method = HF_METHOD_AUTO) {
    params.validate();
    hf_problem pr{};
    pr.nu = params.nu;
    pr.zeta = params.zeta;
    pr.T = params.T;
    pr.jac[0] = jac[0];
    pr.jac[1] = jac[1];
    pr.jac[2] = jac[2];
    pr.with_source = with_source ? 1 : 0;
    pr.method = method;
    detail::check(hf_fused_divergence_blob(detail::thread_context(), &pr, in_path.c_str(), out_path.c_str()),
                  "fused_divergence_blob");
}

// Device-buffer form (the rendered kernel's (n_elements, u, divf) contract, render.hpp:79-80).
inline void fused_divergence_device(const hf_problem& pr, const void* u_dev, void* divf_dev, void* stream = nullptr) {
    detail::check(hf_fused_divergence(&pr, u_dev, divf_dev, stream), "hf_fused_divergence");
}

}  // namespace hexfuse_b200
