// hf_capi.cu -- the C ABI (include/hexfuse_b200.h): validation, operator
// construction, method selection, launches, the pipelined host-buffer path and
// the multi-GPU partition.  Everything here is host code; the kernels live in
// the hf_inst_*.cu units.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/hexfuse_b200.h"
#include "hf_dispatch.cuh"
#include "hf_fr.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

}  // namespace

// the error channel shared with hf_blob.cu
int hf_capi_fail(int code, const std::string& msg) { return fail(code, msg); }

namespace {

int cuda_fail(cudaError_t e, const char* where) {
    return fail(HF_ERUNTIME, std::string(where) + ": " + cudaGetErrorString(e));
}

int64_t ipow64(int64_t b, int e) {
    int64_t r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

// ---------------------------------------------------------------------------------------------
// Operators (operators.hpp:17-74): Gauss-Legendre nodes by Newton iteration from
// Chebyshev guesses with exact symmetrisation; D by barycentric weights with the
// row-sum diagonal.  The reference stops at m = 8 (operators.hpp:18); the same
// construction is used for m = 9 (d = 2, p = 8).
// ---------------------------------------------------------------------------------------------
bool gl_nodes(int m, double* x) {
    if (m < 2 || m > 9) return false;
    for (int i = 0; i < m; ++i) {
        double z = std::cos(M_PI * (i + 0.75) / (m + 0.5));
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = 0.0;
            for (int j = 0; j < m; ++j) {
                const double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * j + 1.0) * z * p1 - j * p2) / (j + 1.0);
            }
            const double dp = m * (z * p0 - p1) / (z * z - 1.0);
            const double z1 = z;
            z = z1 - p0 / dp;
            if (std::fabs(z - z1) < 1e-15) break;
        }
        x[m - 1 - i] = z;
    }
    for (int i = 0; i < m / 2; ++i) {
        const double v = 0.5 * (x[m - 1 - i] - x[i]);
        x[i] = -v;
        x[m - 1 - i] = v;
    }
    if (m % 2 == 1) x[m / 2] = 0.0;
    return true;
}

void derivative_matrix(int m, const double* x, double* D) {
    double wb[16];
    for (int k = 0; k < m; ++k) {
        wb[k] = 1.0;
        for (int j = 0; j < m; ++j)
            if (j != k) wb[k] /= (x[k] - x[j]);
    }
    for (int j = 0; j < m; ++j) {
        double diag = 0.0;
        for (int k = 0; k < m; ++k) {
            if (k == j) continue;
            const double v = (wb[k] / wb[j]) / (x[j] - x[k]);
            D[j * m + k] = v;
            diag -= v;
        }
        D[j * m + j] = diag;
    }
}

struct OpCache {
    double D[10][hfb::kMaxM * hfb::kMaxM];
    double x[10][hfb::kMaxM];
    bool ok[10];
    OpCache() {
        for (int m = 0; m < 10; ++m) {
            double xs[16];
            ok[m] = gl_nodes(m, xs);
            if (ok[m]) {
                derivative_matrix(m, xs, D[m]);
                for (int i = 0; i < m && i < hfb::kMaxM; ++i) x[m][i] = xs[i];
            }
        }
    }
};
const OpCache& ops() {
    static const OpCache c;
    return c;
}

// ---------------------------------------------------------------------------------------------
// Validation (equations.hpp:19-23, layout.hpp:92-99, operators.hpp:18)
// ---------------------------------------------------------------------------------------------
int validate(const hf_problem* pr) {
    if (!pr) return fail(HF_EINVAL, "hf_problem: null");
    if (pr->d != 2 && pr->d != 3) return fail(HF_EINVAL, "hf_problem: d must be 2 or 3");
    const int pmax = (pr->d == 3) ? 7 : 8;
    if (pr->p < 1 || pr->p > pmax)
        return fail(HF_EINVAL, "hf_problem: p must be in [1," + std::to_string(pmax) + "] for d=" +
                                   std::to_string(pr->d));
    if (pr->n_elem < 0) return fail(HF_EINVAL, "hf_problem: n_elem must be >= 0");
    if (pr->group < 1) return fail(HF_EINVAL, "hf_problem: group must be >= 1");
    if (pr->precision != HF_FP32 && pr->precision != HF_FP64)
        return fail(HF_EINVAL, "hf_problem: precision must be HF_FP32 or HF_FP64");
    if (!(pr->nu >= 0.0)) return fail(HF_EINVAL, "PhysParams: nu must be >= 0");
    if (!(pr->zeta > 0.0)) return fail(HF_EINVAL, "PhysParams: zeta must be > 0");
    if (!(pr->T > 0.0)) return fail(HF_EINVAL, "PhysParams: T must be > 0");
    if (pr->method < HF_METHOD_AUTO || pr->method > HF_METHOD_PLANAR_MANAGED)
        return fail(HF_EINVAL, "hf_problem: unknown method");
    if ((pr->method == HF_METHOD_PLANAR || pr->method == HF_METHOD_PLANAR_MANAGED) && pr->d != 3)
        return fail(HF_EINVAL, "planar method: d must be 3");
    const int64_t words = ipow64(pr->p + 1, pr->d) * (1 + pr->d + pr->d * pr->d) * int64_t(pr->group);
    if (words > (int64_t(1) << 31)) return fail(HF_EINVAL, "hf_problem: group too large");
    return HF_OK;
}

// ---------------------------------------------------------------------------------------------
// Selection
// ---------------------------------------------------------------------------------------------

// AUTO takes the measured row of the selection table; an explicit LINES request takes the
// row's measured lines variant too (variant 0 when the row selected another method).
void select_method(const hf_problem* pr, int* method, int* variant) {
    *variant = 0;
    *method = pr->method != HF_METHOD_AUTO ? pr->method : HF_METHOD_LINES;
    for (const hfb::SelRow& r : hfb::kSelect)
        if (r.d == pr->d && r.p == pr->p && r.prec == pr->precision) {
            if (pr->method == HF_METHOD_AUTO) {
                *method = r.method;
                *variant = r.variant;
            } else if (pr->method == HF_METHOD_LINES && r.method == HF_METHOD_LINES) {
                *variant = r.variant;
            }
        }
}

// Restores the caller's current device on every return path of an entry point that
// has to switch devices.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Mesh / partition checks of the FR stages (before anything is launched).
int check_mesh(const hf_problem* pr, const hf_mesh* mesh, const void* ghost_lo, const void* ghost_hi,
               const char* who) {
    if (!mesh) return fail(HF_EINVAL, std::string(who) + ": null mesh");
    const int64_t nz = pr->d == 3 ? mesh->dims[2] : 1;
    if (mesh->dims[0] < 1 || mesh->dims[1] < 1 || nz < 1) return fail(HF_EINVAL, std::string(who) + ": bad mesh dims");
    const int64_t n_mesh = int64_t(mesh->dims[0]) * mesh->dims[1] * nz;
    if (mesh->n_local != pr->n_elem || mesh->e_begin < 0 || mesh->e_begin + mesh->n_local > n_mesh)
        return fail(HF_EINVAL, std::string(who) + ": partition must be n_elem elements inside the mesh");
    if (mesh->n_local < n_mesh) {
        const int64_t layer = pr->d == 3 ? int64_t(mesh->dims[0]) * mesh->dims[1] : mesh->dims[0];
        if (mesh->layer != layer || mesh->e_begin % layer || mesh->n_local % layer || !ghost_lo || !ghost_hi)
            return fail(HF_EINVAL,
                        std::string(who) + ": a partition must be whole element layers with both ghost layers");
    }
    return HF_OK;
}

template <class R>
hfb::Params<R> make_params(const hf_problem* pr, const void* u, void* out, void* ws) {
    hfb::Params<R> p;
    std::memset(&p, 0, sizeof(p));
    const int m = pr->p + 1;
    const double* D = ops().D[m];
    for (int i = 0; i < m * m; ++i) p.D[i] = R(D[i]);
    for (int i = 0; i < m; ++i) p.xg[i] = R(ops().x[m][i]);
    for (int t = 0; t < m; ++t) {  // Lagrange basis at -1, +1 (FR stage 1 fused into the lines kernel)
        double a = 1.0, b = 1.0;
        for (int q = 0; q < m; ++q) {
            if (q == t) continue;
            a *= (-1.0 - ops().x[m][q]) / (ops().x[m][t] - ops().x[m][q]);
            b *= (1.0 - ops().x[m][q]) / (ops().x[m][t] - ops().x[m][q]);
        }
        p.lm[t] = R(a);
        p.lp[t] = R(b);
    }
    const int h = m / 2;
    for (int i = 0; i <= h && i < hfb::kMaxH; ++i) {
        for (int t = 0; t < h; ++t) {
            p.DE[i * hfb::kMaxH + t] = R(0.5 * (D[i * m + t] + D[i * m + (m - 1 - t)]));
            p.DO[i * hfb::kMaxH + t] = R(0.5 * (D[i * m + t] - D[i * m + (m - 1 - t)]));
        }
        p.DC[i] = (m % 2 == 1) ? R(D[i * m + h]) : R(0);
    }
    p.nu = R(pr->nu);
    p.zeta = R(pr->zeta);
    p.invT = R(1.0 / pr->T);
    for (int a = 0; a < 3; ++a) {
        p.jac[a] = R(pr->jac[a]);
        p.jac_invT[a] = R(pr->jac[a] / pr->T);
    }
    p.u = static_cast<const R*>(u);
    p.out = static_cast<R*>(out);
    p.ws = static_cast<R*>(ws);
    p.n_elem = pr->n_elem;
    p.group = pr->group;
    p.group_words = int64_t(pr->group) * ipow64(m, pr->d) * (1 + pr->d + pr->d * pr->d);
    p.total_words = ((pr->n_elem + pr->group - 1) / pr->group) * p.group_words;
    p.fast_ok = 0;
    return p;
}

// FR stage parameters: Lagrange basis at -1/+1 and the DG correction-function
// derivatives g_L'(x_i), g_R'(x_i) (g_L = (-1)^m/2 (P_m - P_{m-1}), g_R(x) = g_L(-x)).
template <class R>
hfb::FrParams<R> make_fr_params(const hf_problem* pr, const hf_mesh* mesh, const void* uf, const void* glo,
                                const void* ghi) {
    hfb::FrParams<R> f;
    std::memset(&f, 0, sizeof(f));
    const int m = pr->p + 1;
    const double* x = ops().x[m];
    for (int t = 0; t < m; ++t) {
        double a = 1.0, b = 1.0;
        for (int q = 0; q < m; ++q) {
            if (q == t) continue;
            a *= (-1.0 - x[q]) / (x[t] - x[q]);
            b *= (1.0 - x[q]) / (x[t] - x[q]);
        }
        f.lm[t] = R(a);
        f.lp[t] = R(b);
    }
    auto gl_deriv = [m](double xx) {
        double p0 = 1.0, p1 = xx, d0 = 0.0, d1 = 1.0, dm1 = 1.0;  // P_n, P_n' recurrences
        for (int n = 2; n <= m; ++n) {
            const double p2 = ((2.0 * n - 1.0) * xx * p1 - (n - 1.0) * p0) / n;
            const double d2 = d0 + (2.0 * n - 1.0) * p1;
            p0 = p1;
            p1 = p2;
            d0 = d1;
            d1 = d2;
            if (n == m - 1) dm1 = d1;
        }
        return ((m % 2 == 0) ? 0.5 : -0.5) * (d1 - dm1);
    };
    for (int i = 0; i < m; ++i) {
        f.gl[i] = R(gl_deriv(x[i]));
        f.gr[i] = R(-gl_deriv(-x[i]));
    }
    if (mesh) {
        for (int a = 0; a < 3; ++a) f.mesh.dims[a] = mesh->dims[a];
        if (pr->d == 2) f.mesh.dims[2] = 1;
        f.mesh.e_begin = mesh->e_begin;
        f.mesh.n_local = mesh->n_local;
        f.mesh.layer = mesh->layer;
    }
    f.uf = static_cast<const R*>(uf);
    f.ghost_lo = static_cast<const R*>(glo);
    f.ghost_hi = static_cast<const R*>(ghi);
    return f;
}

// lines "variant" of the grouped-chunk kernel (LinesShape GS < NE, hf_dispatch.cuh)
constexpr int kGroupedVariant = 100;

// A caller's AoSoA group that is not the selected chunk (e.g. the reference's planar group
// 4*floor(32/m), or a solver's own AoSoA width): the chunk predicted fastest among
//   exact    a one-chunk variant whose chunk is the group (one contiguous range),
//   grouped  NE0 / G whole groups per chunk (a power-of-two group below NE0; contiguous),
//   tile     a strided box of NE elements of one group, one TMA tensor copy per direction,
// scored  fill(G, NE) * rows(NE * w) * occupancy(CTAs per SM), calibrated on B200
// (tools/tile_probe.py, profiles/r02/tile_probe_d3.jsonl): TMA moves a tile box at about
// one row per 3 SM cycles whatever the row length up to 32 B, so 16-byte rows cap a kernel
// near 0.53 of the HBM roofline, 32-byte rows near 0.9, >= 64-byte rows (and contiguous
// chunks) reach it; one resident CTA per SM serialises load, sweeps and store (~0.6); fill
// is the used fraction of the group's sub-chunks (G = 20 in chunks of 16: 20 / 32).  Ties go
// to exact, then grouped, then tile.  Groups whose stride is not a 16-byte multiple and
// match no chunk take the guarded path of the selected chunk size.
template <class R>
int lines_variant_for_group(const hf_problem* pr, int variant, const hfb::Params<R>& prm, bool faces) {
    const int w = int(sizeof(R)), m = pr->p + 1, G = pr->group;
    const int ne0 = hfb::lines_ne0(w, pr->d, m);
    const int ne_sel = hfb::variant_ne_of(ne0, variant);
    if (G == ne_sel) return variant;
    auto available = [&](int v) {
        int rc;
        if constexpr (sizeof(R) == 4)
            rc = pr->d == 3 ? hfb::lines_f32_d3(pr->p, v, false, prm, nullptr, nullptr, true, faces)
                            : hfb::lines_f32_d2(pr->p, v, false, prm, nullptr, nullptr, true, faces);
        else
            rc = pr->d == 3 ? hfb::lines_f64_d3(pr->p, v, false, prm, nullptr, nullptr, true, faces)
                            : hfb::lines_f64_d2(pr->p, v, false, prm, nullptr, nullptr, true, faces);
        return rc == 0;
    };
    const int64_t np = ipow64(m, pr->d), nv = 1 + pr->d + pr->d * pr->d;
    auto occupancy = [&](int ne) {  // shared memory of hf_lines_kernel (LinesShape::SMEM), 228 KB per SM
        const int64_t smem = 128 + ((ne * np * nv * w + 15) / 16 * 16 + 32) + ne * np * (1 + pr->d) * w;
        const int64_t bps = (228 * 1024) / (smem + 1024);
        return bps >= 3 ? 1.0 : bps == 2 ? 0.95 : 0.6;
    };
    int best = -1;
    double best_score = -1.0;
    auto consider = [&](int v, double score) {
        if (score > best_score + 1e-9) {
            best = v;
            best_score = score;
        }
    };
    const int cand[4] = {0, 1, 7, 2};
    for (int v : cand)
        if (hfb::variant_ne_of(ne0, v) == G && available(v)) consider(v, occupancy(G));
    if (!faces && G < ne0 && (G & (G - 1)) == 0 && ne0 % G == 0) {
        int rc;
        if constexpr (sizeof(R) == 4)
            rc = pr->d == 3 ? hfb::lines_grouped_f32_d3(pr->p, G, false, prm, nullptr, nullptr, true)
                            : hfb::lines_grouped_f32_d2(pr->p, G, false, prm, nullptr, nullptr, true);
        else
            rc = pr->d == 3 ? hfb::lines_grouped_f64_d3(pr->p, G, false, prm, nullptr, nullptr, true)
                            : hfb::lines_grouped_f64_d2(pr->p, G, false, prm, nullptr, nullptr, true);
        if (rc == 0) consider(kGroupedVariant, occupancy(ne0));
    }
    if ((int64_t(G) * w) % 16 == 0) {
        for (int v : cand) {
            const int ne = hfb::variant_ne_of(ne0, v);
            if (ne < 1 || ne == G || (ne * w) % 16 != 0 || !available(v)) continue;
            const double fill = double(G) / (double((G + ne - 1) / ne) * ne);
            const int row = ne * w;
            // 32-byte rows: 0.9 of the roofline in bursts, 0.8 relative to 64-byte rows under sustained
            // load (profiles/r02/groups_sustained/: p2 FP32 group 40, NE 16 at 5/6 fill 0.86 against
            // NE 8 full 0.81)
            consider(v, fill * (row >= 64 ? 1.0 : row >= 32 ? 0.8 : 0.53) * occupancy(ne));
        }
    }
    // the tile ring (variant 24, built at d3 p5): 2 NE0 elements in a two-stage TMA ring, so
    // chunk loads and stores overlap the sweeps although the chunk leaves one CTA per SM
    if (!faces && available(hfb::kTileRingVariant)) {
        const int ne = hfb::variant_ne_of(ne0, hfb::kTileRingVariant);
        if (G == ne) {
            consider(hfb::kTileRingVariant, 1.0);
        } else if ((int64_t(G) * w) % 16 == 0 && (ne * w) % 16 == 0 && G % ne == 0) {
            // whole sub-chunks only: with a short last sub-chunk per group (G = 12, 20 at NE = 8)
            // the ring measured 0.40-0.43 against 0.53 for the one-chunk NE0 tile
            // (profiles/r02/tile_ring/groups_p5.jsonl)
            const int row = ne * w;
            consider(hfb::kTileRingVariant, row >= 64 ? 1.0 : row >= 32 ? 0.9 : 0.53);
        }
    }
    if (best >= 0) return best;
    // guarded path (a group that is not a 16-byte stride and no chunk size): every staged word
    // is one cp.async copy, so the contiguous run per row (min(NE, G) words) and the resident
    // CTAs decide -- measured 0.33-0.70 for G = 3, 5, 7, 15 (profiles/r02/groups_odd_*.jsonl)
    double best_g = -1.0;
    for (int v : cand) {
        const int ne = hfb::variant_ne_of(ne0, v);
        if (ne < 1 || !available(v)) continue;
        const double run = std::min(1.0, double(std::min(ne, G)) * w / 64.0);
        const double score = run * occupancy(ne);
        if (score > best_g + 1e-9) {
            best = v;
            best_g = score;
        }
    }
    if (best >= 0) return best;
    return hfb::is_one_chunk_variant(variant) ? variant : 0;
}

// Resolve + launch (dry: describe only).  ws only for the unfused method.
int dispatch(const hf_problem* pr, const void* u, void* out, void* ws, cudaStream_t st, hfb::KInfo* info, bool dry,
             int force_method = -1, int force_variant = -1, bool faces = false, void* uf = nullptr) {
    int method, variant;
    select_method(pr, &method, &variant);
    if (faces && method == HF_METHOD_LINES && hfb::faces_variant_override(pr->d, pr->p) >= 0)
        variant = hfb::faces_variant_override(pr->d, pr->p);
    if (force_method >= 0) method = force_method;
    if (force_variant >= 0) variant = force_variant;
    const bool src = pr->with_source != 0;
    int rc;
    if (faces && method != HF_METHOD_LINES) return hfb::kUnsupported;
    if (pr->precision == HF_FP32) {
        auto prm = make_params<float>(pr, u, out, ws);
        prm.uf = static_cast<float*>(uf);
        if (method == HF_METHOD_LINES && force_variant < 0) variant = lines_variant_for_group(pr, variant, prm, faces);
        if (method == HF_METHOD_LINES && variant == kGroupedVariant)
            rc = pr->d == 3 ? hfb::lines_grouped_f32_d3(pr->p, pr->group, src, prm, st, info, dry)
                            : hfb::lines_grouped_f32_d2(pr->p, pr->group, src, prm, st, info, dry);
        else if (method == HF_METHOD_PLANAR) rc = hfb::planar_f32(pr->p, src, prm, st, info, dry);
        else if (method == HF_METHOD_PLANAR_MANAGED) rc = hfb::planar_managed_f32(pr->p, src, prm, st, info, dry);
        else if (method == HF_METHOD_UNFUSED) rc = hfb::unfused_f32(pr->d, pr->p, src, prm, st, info, dry);
        else rc = pr->d == 3 ? hfb::lines_f32_d3(pr->p, variant, src, prm, st, info, dry, faces)
                             : hfb::lines_f32_d2(pr->p, variant, src, prm, st, info, dry, faces);
    } else {
        auto prm = make_params<double>(pr, u, out, ws);
        prm.uf = static_cast<double*>(uf);
        if (method == HF_METHOD_LINES && force_variant < 0) variant = lines_variant_for_group(pr, variant, prm, faces);
        if (method == HF_METHOD_LINES && variant == kGroupedVariant)
            rc = pr->d == 3 ? hfb::lines_grouped_f64_d3(pr->p, pr->group, src, prm, st, info, dry)
                            : hfb::lines_grouped_f64_d2(pr->p, pr->group, src, prm, st, info, dry);
        else if (method == HF_METHOD_PLANAR) rc = hfb::planar_f64(pr->p, src, prm, st, info, dry);
        else if (method == HF_METHOD_PLANAR_MANAGED) rc = hfb::planar_managed_f64(pr->p, src, prm, st, info, dry);
        else if (method == HF_METHOD_UNFUSED) rc = hfb::unfused_f64(pr->d, pr->p, src, prm, st, info, dry);
        else rc = pr->d == 3 ? hfb::lines_f64_d3(pr->p, variant, src, prm, st, info, dry, faces)
                             : hfb::lines_f64_d2(pr->p, variant, src, prm, st, info, dry, faces);
    }
    if (faces && rc == hfb::kUnsupported) return rc;  // caller falls back to the separate stage-1 kernel
    if (rc == hfb::kUnsupported) return fail(HF_EINVAL, "no kernel for this (method, d, p, variant)");
    if (rc != 0) return cuda_fail(cudaError_t(rc), "kernel launch");
    return HF_OK;
}

size_t word_bytes(const hf_problem* pr) { return pr->precision == HF_FP32 ? 4 : 8; }

// The kernels read u while other CTAs write divf: the two fields must not share a byte.
bool fields_overlap(const hf_problem* pr, const void* u, const void* out) {
    const int64_t gw = int64_t(pr->group) * ipow64(pr->p + 1, pr->d) * (1 + pr->d + pr->d * pr->d);
    const uintptr_t bytes = uintptr_t(((pr->n_elem + pr->group - 1) / pr->group) * gw) * word_bytes(pr);
    const uintptr_t a = reinterpret_cast<uintptr_t>(u), b = reinterpret_cast<uintptr_t>(out);
    return bytes > 0 && a < b + bytes && b < a + bytes;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

const char* hf_last_error(void) { return g_last_error.c_str(); }
const char* hf_version(void) { return "hexfuse_b200 0.1 (sm_100a)"; }

int hf_n_vars(int d) { return (d == 2 || d == 3) ? 1 + d + d * d : -1; }

int hf_validate(const hf_problem* pr) { return validate(pr); }

int64_t hf_field_words(const hf_problem* pr) {
    if (!pr || pr->group < 1 || (pr->d != 2 && pr->d != 3) || pr->n_elem < 0) return -1;
    const int64_t ng = (pr->n_elem + pr->group - 1) / pr->group;
    return ng * pr->group * ipow64(pr->p + 1, pr->d) * (1 + pr->d + pr->d * pr->d);
}

int64_t hf_offset(const hf_problem* pr, int64_t e, int i, int j, int k, int v) {
    const int m = pr->p + 1;
    const int64_t np = ipow64(m, pr->d);
    const int64_t gw = int64_t(pr->group) * np * (1 + pr->d + pr->d * pr->d);
    const int64_t pt = i + int64_t(m) * j + int64_t(m) * m * k;
    return (e / pr->group) * gw + (e % pr->group) + int64_t(pr->group) * (pt + np * v);
}

int hf_derivative_matrix(int m, double* D_out, double* nodes_out) {
    double x[16];
    if (!gl_nodes(m, x)) return fail(HF_EINVAL, "gauss_legendre_points: m must be in [2,9]");
    if (nodes_out) std::memcpy(nodes_out, x, sizeof(double) * m);
    if (D_out) derivative_matrix(m, x, D_out);
    return HF_OK;
}

int64_t hf_algorithmic_bytes_per_point(const hf_problem* pr) {
    return 2 * int64_t(1 + pr->d + pr->d * pr->d) * int64_t(word_bytes(pr));
}

int hf_selected_method(const hf_problem* pr) {
    if (int rc = validate(pr)) return -rc;
    int method, variant;
    select_method(pr, &method, &variant);
    return method;
}

int hf_kernel_info_get(const hf_problem* pr, hf_kernel_info* out) {
    if (int rc = validate(pr)) return rc;
    hfb::KInfo ki;
    if (int rc = dispatch(pr, nullptr, nullptr, nullptr, nullptr, &ki, true)) return rc;
    out->method = ki.method;
    out->elems_per_cta = ki.elems_per_cta;
    out->block_threads = ki.block_threads;
    out->shared_bytes = ki.shared_bytes;
    out->registers = ki.registers;
    out->grid = ki.grid;
    out->bulk_path = ki.bulk_path;
    out->blocks_per_sm = ki.blocks_per_sm;
    std::memcpy(out->name, ki.name, sizeof(out->name));
    return HF_OK;
}

int hf_preferred_group(const hf_problem* pr) {
    if (int rc = validate(pr)) return -rc;
    hf_problem q = *pr;
    int method, variant;
    select_method(pr, &method, &variant);
    if (method == HF_METHOD_UNFUSED) {  // hfb::unfused_group: direction blocks of <= 48 KB, >= 16-byte rows
        const int64_t blk = ipow64(pr->p + 1, pr->d) * (1 + pr->d + pr->d * pr->d) * int64_t(word_bytes(pr));
        int g = 64;
        while (g > 16 / int(word_bytes(pr)) && g * blk > 48 * 1024) g /= 2;
        return g;
    }
    hfb::KInfo ki;  // the selected variant's chunk, whatever pr->group is
    if (dispatch(&q, nullptr, nullptr, nullptr, nullptr, &ki, true, method, variant)) return -HF_EINVAL;
    return ki.elems_per_cta;
}

int hf_fused_divergence(const hf_problem* pr, const void* u_dev, void* divf_dev, void* stream) {
    if (int rc = validate(pr)) return rc;
    int method, variant;
    select_method(pr, &method, &variant);
    if (method == HF_METHOD_UNFUSED)
        return fail(HF_EINVAL, "hf_fused_divergence: use hf_unfused_divergence for the unfused method");
    if (pr->n_elem > 0 && (!u_dev || !divf_dev)) return fail(HF_EINVAL, "hf_fused_divergence: null buffer");
    if (pr->n_elem > 0 && fields_overlap(pr, u_dev, divf_dev))
        return fail(HF_EINVAL, "hf_fused_divergence: in-place not supported (u and divf overlap)");
    return dispatch(pr, u_dev, divf_dev, nullptr, static_cast<cudaStream_t>(stream), nullptr, false);
}

size_t hf_unfused_workspace_bytes(const hf_problem* pr) {
    if (validate(pr)) return 0;
    return size_t(hf_field_words(pr)) * size_t(pr->d) * word_bytes(pr);
}

int64_t hf_face_words(const hf_problem* pr) {
    if (!pr || pr->group < 1 || (pr->d != 2 && pr->d != 3) || pr->n_elem < 0) return -1;
    const int m = pr->p + 1;
    const int64_t ng = (pr->n_elem + pr->group - 1) / pr->group;
    return ng * pr->group * 2 * pr->d * ipow64(m, pr->d - 1) * (1 + pr->d + pr->d * pr->d);
}

int64_t hf_geometry_words(const hf_problem* pr) {
    if (!pr || pr->group < 1 || (pr->d != 2 && pr->d != 3) || pr->n_elem < 0) return -1;
    const int64_t ng = (pr->n_elem + pr->group - 1) / pr->group;
    return ng * pr->group * (int64_t(1) << pr->d) * pr->d;
}

int hf_fused_divergence_mapped(const hf_problem* pr, const void* u_dev, const void* geom_dev, void* divf_dev,
                               void* stream) {
    if (int rc = validate(pr)) return rc;
    if (pr->n_elem > 0 && (!u_dev || !divf_dev || !geom_dev))
        return fail(HF_EINVAL, "hf_fused_divergence_mapped: null buffer");
    if (pr->n_elem > 0 && fields_overlap(pr, u_dev, divf_dev))
        return fail(HF_EINVAL, "hf_fused_divergence_mapped: in-place not supported (u and divf overlap)");
    const bool src = pr->with_source != 0;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    int rc;
    if (pr->precision == HF_FP32) {
        auto prm = make_params<float>(pr, u_dev, divf_dev, nullptr);
        prm.geo = static_cast<const float*>(geom_dev);
        rc = hfb::mapped_f32(pr->d, pr->p, src, prm, st, nullptr, false);
    } else {
        auto prm = make_params<double>(pr, u_dev, divf_dev, nullptr);
        prm.geo = static_cast<const double*>(geom_dev);
        rc = hfb::mapped_f64(pr->d, pr->p, src, prm, st, nullptr, false);
    }
    if (rc == hfb::kUnsupported) return fail(HF_EINVAL, "no mapped kernel for this (d, p)");
    if (rc != 0) return cuda_fail(cudaError_t(rc), "mapped kernel launch");
    return HF_OK;
}

int hf_mapped_kernel_info(const hf_problem* pr, hf_kernel_info* out) {
    if (int rc = validate(pr)) return rc;
    if (!out) return fail(HF_EINVAL, "hf_mapped_kernel_info: null output");
    hfb::KInfo ki;
    const auto dummy_f = make_params<float>(pr, nullptr, nullptr, nullptr);
    const auto dummy_d = make_params<double>(pr, nullptr, nullptr, nullptr);
    const int rc = pr->precision == HF_FP32 ? hfb::mapped_f32(pr->d, pr->p, pr->with_source != 0, dummy_f, nullptr, &ki, true)
                                            : hfb::mapped_f64(pr->d, pr->p, pr->with_source != 0, dummy_d, nullptr, &ki, true);
    if (rc == hfb::kUnsupported) return fail(HF_EINVAL, "no mapped kernel for this (d, p)");
    out->method = ki.method;
    out->elems_per_cta = ki.elems_per_cta;
    out->block_threads = ki.block_threads;
    out->shared_bytes = ki.shared_bytes;
    out->registers = ki.registers;
    out->grid = ki.grid;
    out->bulk_path = ki.bulk_path;
    out->blocks_per_sm = ki.blocks_per_sm;
    std::memcpy(out->name, ki.name, sizeof(out->name));
    return HF_OK;
}

int hf_fr_project(const hf_problem* pr, const void* u_dev, void* uf_dev, void* stream) {
    if (int rc = validate(pr)) return rc;
    if (pr->n_elem > 0 && (!u_dev || !uf_dev)) return fail(HF_EINVAL, "hf_fr_project: null buffer");
    int rc;
    if (pr->precision == HF_FP32) {
        const auto prm = make_params<float>(pr, u_dev, nullptr, nullptr);
        const auto fp = make_fr_params<float>(pr, nullptr, nullptr, nullptr, nullptr);
        rc = hfb::fr_f32(1, pr->d, pr->p, prm, fp, static_cast<float*>(uf_dev), static_cast<cudaStream_t>(stream));
    } else {
        const auto prm = make_params<double>(pr, u_dev, nullptr, nullptr);
        const auto fp = make_fr_params<double>(pr, nullptr, nullptr, nullptr, nullptr);
        rc = hfb::fr_f64(1, pr->d, pr->p, prm, fp, static_cast<double*>(uf_dev), static_cast<cudaStream_t>(stream));
    }
    if (rc < 0) return fail(HF_EINVAL, "hf_fr_project: unsupported (d, p)");
    if (rc != 0) return cuda_fail(cudaError_t(rc), "hf_fr_project launch");
    return HF_OK;
}

int hf_fr_correct(const hf_problem* pr, const hf_mesh* mesh, const void* uf_dev, const void* ghost_lo,
                  const void* ghost_hi, void* divf_dev, void* stream) {
    if (int rc = validate(pr)) return rc;
    if (int rc = check_mesh(pr, mesh, ghost_lo, ghost_hi, "hf_fr_correct")) return rc;
    if (pr->n_elem > 0 && (!uf_dev || !divf_dev)) return fail(HF_EINVAL, "hf_fr_correct: null buffer");
    int rc;
    if (pr->precision == HF_FP32) {
        const auto prm = make_params<float>(pr, nullptr, divf_dev, nullptr);
        const auto fp = make_fr_params<float>(pr, mesh, uf_dev, ghost_lo, ghost_hi);
        rc = hfb::fr_f32(2, pr->d, pr->p, prm, fp, nullptr, static_cast<cudaStream_t>(stream));
    } else {
        const auto prm = make_params<double>(pr, nullptr, divf_dev, nullptr);
        const auto fp = make_fr_params<double>(pr, mesh, uf_dev, ghost_lo, ghost_hi);
        rc = hfb::fr_f64(2, pr->d, pr->p, prm, fp, nullptr, static_cast<cudaStream_t>(stream));
    }
    if (rc < 0) return fail(HF_EINVAL, "hf_fr_correct: unsupported (d, p)");
    if (rc != 0) return cuda_fail(cudaError_t(rc), "hf_fr_correct launch");
    return HF_OK;
}

int hf_fr_divergence_faces(const hf_problem* pr, const void* u_dev, void* uf_dev, void* divf_dev, void* stream) {
    if (int rc = validate(pr)) return rc;
    if (pr->n_elem > 0 && (!u_dev || !uf_dev || !divf_dev))
        return fail(HF_EINVAL, "hf_fr_divergence_faces: null buffer");
    if (pr->n_elem > 0 && fields_overlap(pr, u_dev, divf_dev))
        return fail(HF_EINVAL, "hf_fr_divergence_faces: in-place not supported (u and divf overlap)");
    // stages 1+2+3+6 in one pass of the lines kernel (faces written beside the divergence);
    // the separate stage-1 kernel where no fused form is built (e.g. a planar selection)
#ifdef HF_FACES_AB
    const char* fv = std::getenv("HF_FACES_VARIANT");
    const int force_v = fv ? std::atoi(fv) : -1;
#else
    const int force_v = -1;
#endif
    const int rc = dispatch(pr, u_dev, divf_dev, nullptr, static_cast<cudaStream_t>(stream), nullptr, false, -1,
                            force_v, true, uf_dev);
    if (rc == hfb::kUnsupported) {
        if (int r2 = hf_fused_divergence(pr, u_dev, divf_dev, stream)) return r2;  // stages 2+3+6
        return hf_fr_project(pr, u_dev, uf_dev, stream);                         // stage 1
    }
    return rc;
}

int hf_fr_residual(const hf_problem* pr, const int* dims, const void* u_dev, void* uf_dev, void* divf_dev,
                   void* stream) {
    if (!dims) return fail(HF_EINVAL, "hf_fr_residual: null dims");
    hf_mesh ms{};
    ms.dims[0] = dims[0];
    ms.dims[1] = dims[1];
    ms.dims[2] = pr && pr->d == 3 ? dims[2] : 1;
    ms.e_begin = 0;
    ms.n_local = pr ? pr->n_elem : 0;
    ms.layer = 0;
    if (int rc = validate(pr)) return rc;
    if (ms.dims[0] < 1 || ms.dims[1] < 1 || ms.dims[2] < 1 || int64_t(ms.dims[0]) * ms.dims[1] * ms.dims[2] != pr->n_elem)
        return fail(HF_EINVAL, "hf_fr_residual: dims must be >= 1 with product n_elem");
    if (int rc = check_mesh(pr, &ms, nullptr, nullptr, "hf_fr_residual")) return rc;  // before any launch
    if (pr->n_elem > 0 && (!u_dev || !uf_dev || !divf_dev)) return fail(HF_EINVAL, "hf_fr_residual: null buffer");
    if (pr->n_elem > 0 && fields_overlap(pr, u_dev, divf_dev))
        return fail(HF_EINVAL, "hf_fr_residual: in-place not supported (u and divf overlap)");
    // Where measured faster (hfb::fr_residual_fused): stage 1 (the faces), then ONE lines kernel
    // for stages 2+3+6 and 4+5 -- the residual leaves shared memory once (hf_lines_fr_kernel).
    // Elsewhere the pair: stages 1+2+3+6 in the lines kernel, then the correction kernel.
    static const int forced = [] {  // HF_FR_FUSED=0 / 1 forces the pair / the one-pass form (A/B runs)
        const char* e = std::getenv("HF_FR_FUSED");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    bool fused = forced == 1;
    if (forced < 0) {
        const auto prm0 = make_params<float>(pr, nullptr, nullptr, nullptr);
        const auto prm1 = make_params<double>(pr, nullptr, nullptr, nullptr);
        fused = (pr->precision == HF_FP32 ? hfb::fr_f32(5, pr->d, pr->p, prm0, hfb::FrParams<float>{}, nullptr, nullptr)
                                          : hfb::fr_f64(5, pr->d, pr->p, prm1, hfb::FrParams<double>{}, nullptr, nullptr)) == 1;
    }
    if (fused && pr->n_elem > 0) {
        if (int rc = hf_fr_project(pr, u_dev, uf_dev, stream)) return rc;  // stage 1
        int rc;
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int which = pr->with_source ? 4 : 3;
        if (pr->precision == HF_FP32) {
            const auto prm = make_params<float>(pr, u_dev, divf_dev, nullptr);
            const auto fp = make_fr_params<float>(pr, &ms, uf_dev, nullptr, nullptr);
            rc = hfb::fr_f32(which, pr->d, pr->p, prm, fp, nullptr, st);
        } else {
            const auto prm = make_params<double>(pr, u_dev, divf_dev, nullptr);
            const auto fp = make_fr_params<double>(pr, &ms, uf_dev, nullptr, nullptr);
            rc = hfb::fr_f64(which, pr->d, pr->p, prm, fp, nullptr, st);
        }
        if (rc == 0) return HF_OK;
        if (rc > 0) return cuda_fail(cudaError_t(rc), "hf_fr_residual: fused stages 2-6");
        // no fused form for this (d, p): stages 2+3+6, then 4+5 (the faces are written)
        if (int r2 = hf_fused_divergence(pr, u_dev, divf_dev, stream)) return r2;
        return hf_fr_correct(pr, &ms, uf_dev, nullptr, nullptr, divf_dev, stream);
    }
    if (int rc = hf_fr_divergence_faces(pr, u_dev, uf_dev, divf_dev, stream)) return rc;  // stages 1+2+3+6
    return hf_fr_correct(pr, &ms, uf_dev, nullptr, nullptr, divf_dev, stream);  // stages 4+5
}

int hf_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return fail(HF_EINVAL, "hf_ipc_handle: null argument");
    // the handle names the whole allocation (caching allocators hand out pieces of one)
    // (driver entry point through the runtime: no link-time dependency on libcuda)
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<GetRange>(fn);
    }();
    CUdeviceptr base = 0;
    size_t size = 0;
    if (!get_range || get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return fail(HF_ERUNTIME, "hf_ipc_handle: cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == HF_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = int64_t(reinterpret_cast<uintptr_t>(dev_ptr) - uintptr_t(base));
    return HF_OK;
}

int hf_ipc_open(const void* handle, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return fail(HF_EINVAL, "hf_ipc_open: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    return HF_OK;
}

int hf_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return HF_OK;
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
    return HF_OK;
}

int hf_unfused_divergence(const hf_problem* pr, const void* u_dev, void* divf_dev, void* ws_dev, void* stream) {
    if (int rc = validate(pr)) return rc;
    if (pr->n_elem > 0 && (!u_dev || !divf_dev || !ws_dev)) return fail(HF_EINVAL, "hf_unfused_divergence: null buffer");
    return dispatch(pr, u_dev, divf_dev, ws_dev, static_cast<cudaStream_t>(stream), nullptr, false,
                    HF_METHOD_UNFUSED, 0);
}

// Internal hook for tuning sweeps (tools/select_methods.py): launch a specific
// method/variant regardless of the selection table.  Not part of the header.
HF_API int hf_fused_divergence_variant(const hf_problem* pr, int method, int variant, const void* u_dev, void* divf_dev,
                                void* stream, hf_kernel_info* info) {
    if (int rc = validate(pr)) return rc;
    hfb::KInfo ki;
    int rc = dispatch(pr, u_dev, divf_dev, nullptr, static_cast<cudaStream_t>(stream), &ki, info != nullptr && !u_dev,
                      method, variant);
    if (rc) return rc;
    if (info) {
        if (u_dev) {
            hfb::KInfo k2;
            dispatch(pr, nullptr, nullptr, nullptr, nullptr, &k2, true, method, variant);
            ki = k2;
        }
        info->method = ki.method;
        info->elems_per_cta = ki.elems_per_cta;
        info->block_threads = ki.block_threads;
        info->shared_bytes = ki.shared_bytes;
        info->registers = ki.registers;
        info->grid = ki.grid;
        info->bulk_path = ki.bulk_path;
        info->blocks_per_sm = ki.blocks_per_sm;
        std::memcpy(info->name, ki.name, sizeof(info->name));
    }
    return HF_OK;
}

int hf_partition(const hf_problem* pr, int n_parts, int part, int64_t* e_begin, int64_t* n_elem_part,
                 int64_t* word_offset) {
    if (int rc = validate(pr)) return rc;
    if (n_parts < 1 || part < 0 || part >= n_parts) return fail(HF_EINVAL, "hf_partition: bad part");
    const int64_t ng = (pr->n_elem + pr->group - 1) / pr->group;
    const int64_t g0 = ng * part / n_parts, g1 = ng * (part + 1) / n_parts;
    const int64_t e0 = g0 * pr->group;
    const int64_t e1 = std::min<int64_t>(pr->n_elem, g1 * pr->group);
    *e_begin = e0;
    *n_elem_part = std::max<int64_t>(0, e1 - e0);
    const int64_t gw = int64_t(pr->group) * ipow64(pr->p + 1, pr->d) * (1 + pr->d + pr->d * pr->d);
    *word_offset = g0 * gw;
    return HF_OK;
}

}  // extern "C"

// =============================================================================================
// Host-buffer path: slices of whole groups streamed through the GPU, H2D / kernel / D2H on
// three rotating streams so both copy engines and the SMs are busy at once.
// =============================================================================================
struct hf_context {
    int device = 0;
    static constexpr int kSlots = 3;
    cudaStream_t stream[kSlots] = {};
    cudaEvent_t done[kSlots] = {};
    void* d_in[kSlots] = {};
    void* d_out[kSlots] = {};
    size_t slot_bytes = 0;
};

namespace {

int ctx_reserve(hf_context* c, size_t bytes) {
    if (bytes <= c->slot_bytes) return HF_OK;
    for (int s = 0; s < hf_context::kSlots; ++s) {
        if (c->d_in[s]) cudaFree(c->d_in[s]);
        if (c->d_out[s]) cudaFree(c->d_out[s]);
        c->d_in[s] = c->d_out[s] = nullptr;
    }
    c->slot_bytes = 0;
    for (int s = 0; s < hf_context::kSlots; ++s) {
        cudaError_t e = cudaMalloc(&c->d_in[s], bytes);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_out[s], bytes);
        if (e != cudaSuccess) return cuda_fail(e, "hf_context: cudaMalloc");
    }
    c->slot_bytes = bytes;
    return HF_OK;
}

// Base slice of the host path: 48 MB (HF_HOST_SLICE_MB overrides it, for tools/host_probe.py).
int64_t host_slice_bytes() {
    static const int64_t b = [] {
        const char* v = std::getenv("HF_HOST_SLICE_MB");
        const long mb = v ? std::atol(v) : 0;
        return int64_t(mb > 0 ? mb : 48) << 20;
    }();
    return b;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

hf_context* hf_context_create(int device) {
    auto* c = new (std::nothrow) hf_context;
    if (!c) return nullptr;
    c->device = device;
    DeviceGuard guard;
    cudaError_t e = cudaSetDevice(device);
    for (int s = 0; s < hf_context::kSlots && e == cudaSuccess; ++s) {
        e = cudaStreamCreateWithFlags(&c->stream[s], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->done[s], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        cuda_fail(e, "hf_context_create");
        hf_context_destroy(c);
        return nullptr;
    }
    return c;
}

void hf_context_destroy(hf_context* c) {
    if (!c) return;
    DeviceGuard guard;
    cudaSetDevice(c->device);
    for (int s = 0; s < hf_context::kSlots; ++s) {
        if (c->stream[s]) cudaStreamSynchronize(c->stream[s]);
        if (c->d_in[s]) cudaFree(c->d_in[s]);
        if (c->d_out[s]) cudaFree(c->d_out[s]);
        if (c->done[s]) cudaEventDestroy(c->done[s]);
        if (c->stream[s]) cudaStreamDestroy(c->stream[s]);
    }
    delete c;
}

int hf_fused_divergence_host(hf_context* c, const hf_problem* pr, const void* u_host, void* divf_host) {
    return hf_fused_divergence_host_batch(c, 1, pr, &u_host, &divf_host);
}

int hf_fused_divergence_host_batch(hf_context* c, int n_fields, const hf_problem* prs, const void* const* u_hosts,
                                   void* const* divf_hosts) {
    if (!c) return fail(HF_EINVAL, "hf_fused_divergence_host: null context");
    if (n_fields < 0 || (n_fields > 0 && (!prs || !u_hosts || !divf_hosts)))
        return fail(HF_EINVAL, "hf_fused_divergence_host_batch: null arrays");
    for (int i = 0; i < n_fields; ++i) {
        if (int rc = validate(&prs[i])) return rc;
        if (prs[i].n_elem > 0 && (!u_hosts[i] || !divf_hosts[i]))
            return fail(HF_EINVAL, "hf_fused_divergence_host: null buffer");
    }
    // in place (u_host == divf_host) is fine: slices are disjoint and each slice's D2H lands
    // after its own H2D; any other overlap between an input and an output is rejected
    for (int i = 0; i < n_fields; ++i)
        for (int j = 0; j < n_fields; ++j) {
            if (prs[i].n_elem == 0 || prs[j].n_elem == 0 || (i == j && u_hosts[i] == divf_hosts[i])) continue;
            const auto* a = static_cast<const unsigned char*>(u_hosts[i]);
            const auto* b = static_cast<const unsigned char*>(divf_hosts[j]);
            const size_t na = size_t(hf_field_words(&prs[i])) * word_bytes(&prs[i]);
            const size_t nb = size_t(hf_field_words(&prs[j])) * word_bytes(&prs[j]);
            if (a < b + nb && b < a + na)
                return fail(HF_EINVAL, "hf_fused_divergence_host_batch: an input overlaps an output");
        }
    DeviceGuard guard;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

    // One slice plan over all fields: slices of whole groups of one field, multiples of
    // the kernel's chunk, at most ~48 MB (the slot size).  The copy pipeline moves one
    // direction alone while it fills (the first H2D) and drains (the last D2H), so the
    // plan ramps up at the start of the first field and down at the end of the last one
    // (b/8, b/4, b/2, b, ..., b, b/2, b/4, b/8); the fields in between stream at full
    // slices with no fill or drain of their own.
    struct Slice {
        int field;
        int64_t g0, ng;
    };
    std::vector<Slice> plan;
    size_t slot_need = 0;
    for (int i = 0; i < n_fields; ++i) {
        const hf_problem* pr = &prs[i];
        if (pr->n_elem == 0) continue;
        const size_t w = word_bytes(pr);
        const int64_t gw = int64_t(pr->group) * ipow64(pr->p + 1, pr->d) * (1 + pr->d + pr->d * pr->d);
        const int64_t n_groups = (pr->n_elem + pr->group - 1) / pr->group;
        int pref = hf_preferred_group(pr);
        if (pref < 1) pref = 1;
        const int64_t chunk_groups = std::max<int64_t>(1, (pref + pr->group - 1) / pr->group);
        auto rnd = [&](int64_t x) { return std::max<int64_t>(chunk_groups, x / chunk_groups * chunk_groups); };
        const int64_t base = std::min<int64_t>(rnd(host_slice_bytes() / int64_t(gw * w)), n_groups);
        const bool up = plan.empty();
        bool down = true;  // the last field with elements ramps down
        for (int k = i + 1; k < n_fields; ++k) down = down && prs[k].n_elem == 0;
        std::vector<int64_t> q;
        const int64_t ramp[3] = {rnd(base / 8), rnd(base / 4), rnd(base / 2)};
        const int64_t tail = ramp[0] + ramp[1] + ramp[2];
        int64_t rem = n_groups;
        const int64_t need = (up ? tail : 0) + (down ? tail : 0) + base;
        if (rem <= need) {  // small: ~6 equal slices (or whole base slices between ramps)
            const int64_t s = (up || down) ? rnd(std::max<int64_t>(1, rem / 6)) : base;
            while (rem > 0) {
                q.push_back(std::min(s, rem));
                rem -= q.back();
            }
        } else {
            if (up)
                for (int k = 0; k < 3; ++k) {
                    q.push_back(ramp[k]);
                    rem -= ramp[k];
                }
            const int64_t end = down ? tail : 0;
            while (rem > end + base) {
                q.push_back(base);
                rem -= base;
            }
            const int64_t mid = (rem - end) / chunk_groups * chunk_groups;  // whole chunks
            if (mid > 0) q.push_back(mid);
            if (down)
                for (int k = 2; k >= 0; --k) q.push_back(ramp[k]);
            q.back() += rem - end - mid;  // the remainder rides in the final slice
        }
        int64_t g0 = 0;
        for (int64_t ng : q) {
            plan.push_back({i, g0, ng});
            g0 += ng;
            slot_need = std::max(slot_need, size_t(ng * gw) * w);
        }
    }
    if (plan.empty()) return HF_OK;
    if (int rc = ctx_reserve(c, slot_need)) return rc;

    // Pageable host memory is pinned for the duration of the call.
    // (Read-only registration needs device support, cudaDevAttrHostRegisterReadOnlySupported:
    // where it is refused the input is registered read-write.  If registration fails
    // altogether, the copies stage through the driver's pageable path -- slower, same result.)
    std::vector<const void*> reg;
    // read-only registration only where the device supports it (otherwise the driver refuses it
    // and the copy falls back to a read-write registration below)
    int ro_ok = 0;
    if (cudaDeviceGetAttribute(&ro_ok, cudaDevAttrHostRegisterReadOnlySupported, c->device) != cudaSuccess) {
        cudaGetLastError();
        ro_ok = 0;
    }
    auto pin = [&](const void* p, size_t bytes, unsigned flags) {
        if (is_pinned(p)) return;
        if (!ro_ok) flags &= ~unsigned(cudaHostRegisterReadOnly);
        if (cudaHostRegister(const_cast<void*>(p), bytes, flags) == cudaSuccess) {
            reg.push_back(p);
            return;
        }
        cudaGetLastError();
        if (flags != cudaHostRegisterDefault &&
            cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterDefault) == cudaSuccess)
            reg.push_back(p);
        else
            cudaGetLastError();
    };
    for (int i = 0; i < n_fields; ++i) {
        if (prs[i].n_elem == 0) continue;
        const size_t total = size_t(hf_field_words(&prs[i])) * word_bytes(&prs[i]);
        if (u_hosts[i] != divf_hosts[i]) pin(u_hosts[i], total, cudaHostRegisterReadOnly);
        pin(divf_hosts[i], total, cudaHostRegisterDefault);  // in place: one read-write registration
    }

    int rc = HF_OK;
    for (size_t s_idx = 0; s_idx < plan.size() && rc == HF_OK; ++s_idx) {
        const Slice& sl = plan[s_idx];
        const hf_problem* pr = &prs[sl.field];
        const size_t w = word_bytes(pr);
        const int64_t gw = int64_t(pr->group) * ipow64(pr->p + 1, pr->d) * (1 + pr->d + pr->d * pr->d);
        const int slot = int(s_idx % hf_context::kSlots);
        const size_t bytes = size_t(sl.ng * gw) * w;
        cudaStream_t st = c->stream[slot];
        const auto* src = static_cast<const unsigned char*>(u_hosts[sl.field]) + size_t(sl.g0 * gw) * w;
        auto* dst = static_cast<unsigned char*>(divf_hosts[sl.field]) + size_t(sl.g0 * gw) * w;
        // the stream is in-order, so the slot's previous D2H has completed before this H2D lands
        if ((e = cudaMemcpyAsync(c->d_in[slot], src, bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess) {
            rc = cuda_fail(e, "H2D");
            break;
        }
        hf_problem sp = *pr;
        sp.n_elem = std::min<int64_t>(pr->n_elem - sl.g0 * pr->group, sl.ng * pr->group);
        if (sp.method == HF_METHOD_UNFUSED) sp.method = HF_METHOD_AUTO;
        if (sp.n_elem < sl.ng * pr->group) {
            // partial last group: padding comes back as zeros, like the reference's zeroed result (oracle.hpp:26-27)
            if ((e = cudaMemsetAsync(c->d_out[slot], 0, bytes, st)) != cudaSuccess) {
                rc = cuda_fail(e, "memset");
                break;
            }
        }
        rc = dispatch(&sp, c->d_in[slot], c->d_out[slot], nullptr, st, nullptr, false);
        if (rc) break;
        if ((e = cudaMemcpyAsync(dst, c->d_out[slot], bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess) {
            rc = cuda_fail(e, "D2H");
            break;
        }
    }
    for (int s = 0; s < hf_context::kSlots; ++s) {
        e = cudaStreamSynchronize(c->stream[s]);
        if (e != cudaSuccess && rc == HF_OK) rc = cuda_fail(e, "hf_fused_divergence_host");
    }
    for (const void* p : reg) cudaHostUnregister(const_cast<void*>(p));
    return rc;
}

}  // extern "C"
