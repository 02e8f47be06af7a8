"""Generate tests/golden/*.npz from the REFERENCE itself.

Runs hexfuse::random_field / tgv_field / oracle_divergence /
gauss_legendre_points / derivative_matrix compiled in place from
/root/reference/proj/include (oracle/_ref/libhexfuse_ref.so, built by
oracle/Makefile) and stores inputs and outputs as small compressed fixtures.
The fixtures travel with the repo; /root/reference does not exist on the GPU
box, so the GPU tests read only these files.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

PAR = (1.0 / 1600.0, 2.5, 1.0)      # acceptance.cpp:52
PAR_B = (3e-3, 2.5, 1.0)            # test_oracle.cpp:135

# (name, d, p, n_elem, group, fp32, seed, params, jac, with_source)
CASES = []
for p in range(1, 8):
    CASES.append((f"d3_p{p}_fp64", 3, p, 3, 2, False, 2024 + p, PAR, (1.0, 1.0, 1.0), False))
    CASES.append((f"d3_p{p}_fp64_src_jac", 3, p, 2, 1, False, 100 + 10 * p, PAR_B, (1.0, 0.5, 2.0), True))
    CASES.append((f"d3_p{p}_fp32", 3, p, 3, 4, True, 7 + p, PAR, (1.0, 1.0, 1.0), p % 2 == 0))
for p in range(1, 8):
    CASES.append((f"d2_p{p}_fp32", 2, p, 5, 4, True, 300 + p, PAR, (1.0, 1.0, 0.0), p % 2 == 1))
    CASES.append((f"d2_p{p}_fp64_src_jac", 2, p, 3, 2, False, 3, PAR_B, (1.0, 2.0, 0.0), True))


def main():
    if not O.ref_available():
        O.build()
    manifest = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libhexfuse_ref.so "
                "(hexfuse headers from /root/reference/proj/include, compiled in place)", "cases": []}
    arrays = {}
    for (name, d, p, n, g, fp32, seed, par, jac, src) in CASES:
        U = O.ref_random_field(d, p, n, g, fp32, seed)
        out = O.ref_oracle_divergence(d, p, n, g, fp32, U, *par, jac, src)
        arrays[name + "__U"] = U.astype(np.float32) if fp32 else U
        arrays[name + "__out"] = out
        manifest["cases"].append({"name": name, "d": d, "p": p, "n_elem": n, "group": g, "fp32": fp32,
                                  "seed": seed, "nu": par[0], "zeta": par[1], "T": par[2], "jac": list(jac),
                                  "with_source": src,
                                  "sha256_U": hashlib.sha256(U.tobytes()).hexdigest()[:16],
                                  "sha256_out": hashlib.sha256(out.tobytes()).hexdigest()[:16]})
    # vortex fixture (verify.hpp:85-91): factor3(n) brick, width 2, zero-mean pressure
    for (p, n, g, fp32) in [(3, 8, 4, False), (5, 6, 2, False), (2, 12, 4, True)]:
        name = f"tgv_p{p}_{'fp32' if fp32 else 'fp64'}"
        U = O.ref_tgv_field(p, n, g, fp32)
        out = O.ref_oracle_divergence(3, p, n, g, fp32, U, *PAR, (1.0, 1.0, 1.0), False)
        arrays[name + "__U"] = U
        arrays[name + "__out"] = out
        manifest["cases"].append({"name": name, "d": 3, "p": p, "n_elem": n, "group": g, "fp32": fp32, "tgv": True,
                                  "nu": PAR[0], "zeta": PAR[1], "T": PAR[2], "jac": [1.0, 1.0, 1.0],
                                  "with_source": False})
    # operators (operators.hpp:17-74)
    for m in range(2, 9):
        x, D = O.ref_gl_derivative(m)
        arrays[f"gl_nodes_m{m}"] = x
        arrays[f"gl_D_m{m}"] = D
    np.savez_compressed(os.path.join(HERE, "reference_fixtures.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", len(manifest["cases"]), "cases")


if __name__ == "__main__":
    main()
