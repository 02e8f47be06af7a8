// dropin_parity.cpp -- the drop-in demonstration: a C++ program written against
// the REFERENCE's own API (hexfuse::random_field / tgv_field / oracle_divergence
// / field_rel_error / verify_tolerance, /root/reference/proj/include) that swaps
// in hexfuse_b200::fused_divergence_b200 and checks it with the reference's own
// verification metric (verify.hpp:19-35) at the north-star tolerances
// (1e-12 FP64, 1e-5 FP32).  Test infrastructure: built by oracle/Makefile into
// oracle/_ref/dropin_parity (needs the reference headers at build time only),
// run by tests/test_gpu_dropin.py on the GPU box.
#include <hexfuse/oracle.hpp>
#include <hexfuse/verify.hpp>

#include <cstdio>

#include "hexfuse_b200.hpp"

using namespace hexfuse;

int main() {
    const PhysParams par{1.0 / 1600.0, 2.5, 1.0};  // acceptance.cpp:52
    int failures = 0;
    for (Precision prec : {Precision::fp64, Precision::fp32}) {
        for (int p = 1; p <= 7; ++p) {
            for (int block : {128, 256}) {
                ElementConfig cfg;
                cfg.p = p;
                cfg.n_elem = 257;
                cfg.block_threads = block;
                cfg.precision = prec;
                cfg.method = Method::PlanarUnmanaged;  // group = elems_per_block() of the reference planar kernel
                for (int t = 0; t < 2; ++t) {
                    const StateField U = random_field(cfg, 2024 + t);  // seed 2024 (acceptance.cpp:46)
                    const bool src = t == 1;
                    const std::array<double, 3> jac = t == 0 ? std::array<double, 3>{1, 1, 1}
                                                             : std::array<double, 3>{1.0, 0.5, 2.0};
                    const StateField ref = oracle_divergence(U, par, jac, src);
                    const StateField got = hexfuse_b200::fused_divergence_b200(U, par, jac, src);
                    const double err = field_rel_error(got, ref);
                    const double tol = prec == Precision::fp32 ? 1e-5 : 1e-12;
                    const bool ok = err <= tol && got.group == U.group && got.data.size() == U.data.size();
                    std::printf("%s p=%d group=%d src=%d err=%.3e %s\n", to_string(prec), p, U.group, int(src), err,
                                ok ? "ok" : "FAIL");
                    failures += ok ? 0 : 1;
                }
            }
        }
    }
    // the deterministic vortex fixture (verify.hpp:85-91)
    ElementConfig cfg;
    cfg.p = 4;
    cfg.n_elem = 64;
    cfg.precision = Precision::fp64;
    TgvGrid grid;
    grid.elems = factor3(cfg.n_elem);
    const StateField U = tgv_field(cfg, grid, 1.4, 0.08, true);
    const double err = field_rel_error(hexfuse_b200::fused_divergence_b200(U, par, {1, 1, 1}, false),
                                       oracle_divergence(U, par, {1, 1, 1}, false));
    std::printf("tgv p=4 err=%.3e %s\n", err, err <= 1e-12 ? "ok" : "FAIL");
    failures += err <= 1e-12 ? 0 : 1;
    // every reference kernel method (layout.hpp:18) through method_of(): planar, managed planar, lines
    for (Method m : {Method::PlanarUnmanaged, Method::PlanarManaged, Method::Lines}) {
        for (Precision prec : {Precision::fp64, Precision::fp32}) {
            for (int p : {2, 5, 7}) {
                ElementConfig c;
                c.p = p;
                c.n_elem = 97;
                c.precision = prec;
                c.method = m;
                if (m == Method::Lines) c.block_threads = 2 * (p + 1) * (p + 1);  // layout.hpp: n*(p+1)^2
                const StateField U = random_field(c, 99 + p);
                const double e = field_rel_error(
                    hexfuse_b200::fused_divergence_b200(U, par, {1.0, 2.0, 0.5}, true, hexfuse_b200::method_of(m)),
                    oracle_divergence(U, par, {1.0, 2.0, 0.5}, true));
                const double tol = prec == Precision::fp32 ? 1e-5 : 1e-12;
                std::printf("method=%s %s p=%d err=%.3e %s\n", to_string(m), to_string(prec), p, e,
                            e <= tol ? "ok" : "FAIL");
                failures += e <= tol ? 0 : 1;
            }
        }
    }
    // state blobs (layout.hpp:155-200): the reference's export_blob read back through the B200
    // library bit-exactly, a blob-in / blob-out divergence read by the reference's import_blob,
    // and the B200 library's export byte-identical to the reference's
    for (Precision prec : {Precision::fp64, Precision::fp32}) {
        ElementConfig c;
        c.p = 3;
        c.n_elem = 45;
        c.block_threads = 128;
        c.precision = prec;
        c.method = Method::PlanarUnmanaged;
        const StateField U = random_field(c, 31);
        const std::string a = "/tmp/hexfuse_b200_dropin_a.bin", b = "/tmp/hexfuse_b200_dropin_b.bin",
                          r = "/tmp/hexfuse_b200_dropin_r.bin";
        export_blob(U, a);
        const StateField V = hexfuse_b200::import_blob_b200<StateField>(a);
        bool same = V.d == U.d && V.p == U.p && V.n_elem == U.n_elem && V.group == U.group &&
                    V.precision == U.precision && V.data == U.data;
        hexfuse_b200::fused_divergence_blob(a, b, par, {1.0, 0.5, 2.0}, true);
        const StateField out = import_blob(b);
        const double e = field_rel_error(out, oracle_divergence(U, par, {1.0, 0.5, 2.0}, true));
        hexfuse_b200::export_blob_b200(U, r);
        auto slurp = [](const std::string& f) {
            std::FILE* h = std::fopen(f.c_str(), "rb");
            std::string t;
            char buf[4096];
            size_t n;
            while (h && (n = std::fread(buf, 1, sizeof buf, h)) > 0) t.append(buf, n);
            if (h) std::fclose(h);
            return t;
        };
        same = same && slurp(a) == slurp(r) && slurp(a + ".json") == slurp(r + ".json");
        const double tol = prec == Precision::fp32 ? 1e-5 : 1e-12;
        std::printf("blob %s import/export %s, divergence err=%.3e %s\n", to_string(prec), same ? "bit-exact" : "DIFFER",
                    e, same && e <= tol ? "ok" : "FAIL");
        failures += same && e <= tol ? 0 : 1;
    }
    // error mapping: invalid params -> std::invalid_argument, like the reference
    try {
        hexfuse_b200::fused_divergence_b200(U, PhysParams{-1.0, 2.5, 1.0}, {1, 1, 1}, false);
        std::printf("invalid params accepted FAIL\n");
        ++failures;
    } catch (const std::invalid_argument&) {
        std::printf("invalid params -> invalid_argument ok\n");
    }
    std::printf("%s\n", failures == 0 ? "DROPIN PASS" : "DROPIN FAIL");
    return failures == 0 ? 0 : 1;
}
