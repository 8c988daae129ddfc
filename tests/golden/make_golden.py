"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libsglref.so, compiled from
/root/reference/proj/core by oracle/Makefile with the quadrature shim) -- so it
only runs in the build container, where /root/reference exists.  The fixtures
travel with the repo; nothing at test time reads /root/reference.

Fixtures (raw interleaved f64 LE, the reference's vector format,
tools/commands.cpp:194-226):
  rt_B{B}_coeffs.bin   random coefficients, the acceptance suite's draw
                       (mt19937_64 top-53-bit map, acceptance_main.cpp:50-63),
                       seed 1000 + 10 B (criterion 2's first instance, :127)
  rt_B{B}_grid.bin     reference ifsglft of those coefficients
  rt_B{B}_back.bin     reference fsglft of that grid
  mat_B2_forward.bin   reference fsglft of every unit sample vector at B = 2
                       (matrix semantics, test_sgl_transform.cpp:303-346),
                       column-major [psi][omega]
  basis_B3_210.bin     reference ifsglft of the unit coefficient omega(2,1,0)
                       at B = 3 (test_sgl_transform.cpp:205-214)
  manifest.json        sizes, seeds and sha256 of every file

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import Oracle, Reference, coefficient_count, omega_index, sample_count  # noqa: E402

SIZES = (2, 4, 8, 16)


def write(name: str, arr: np.ndarray, manifest: dict, **meta):
    a = np.ascontiguousarray(arr, dtype=np.complex128)
    path = os.path.join(HERE, name)
    a.tofile(path)
    with open(path, "rb") as f:
        digest = hashlib.sha256(f.read()).hexdigest()
    manifest[name] = dict(complex_values=int(a.size), sha256=digest, **meta)


def main():
    manifest = {"generator": "tests/golden/make_golden.py",
                "reference": "oracle/_ref/libsglref.so built from /root/reference/proj/core (quadrature shim)",
                "format": "interleaved float64 little-endian complex (tools/commands.cpp:194-226)"}
    for B in SIZES:
        ref = Reference(B)
        seed = 1000 + 10 * B
        c = Oracle.random_coefficients(B, seed)
        g = ref.inverse(c, threads=1)
        back = ref.forward(g, threads=1)
        write(f"rt_B{B}_coeffs.bin", c, manifest, B=B, seed=seed, what="acceptance-suite coefficients")
        write(f"rt_B{B}_grid.bin", g, manifest, B=B, what="reference ifsglft(coeffs)")
        write(f"rt_B{B}_back.bin", back, manifest, B=B, what="reference fsglft(grid)")
    B = 2
    ref = Reference(B)
    cols = []
    for p in range(sample_count(B)):
        e = np.zeros(sample_count(B), dtype=np.complex128)
        e[p] = 1.0
        cols.append(ref.forward(e, threads=1))
    write("mat_B2_forward.bin", np.stack(cols), manifest, B=2, what="reference fsglft of unit samples, [psi][omega]")
    B = 3
    ref = Reference(B)
    u = np.zeros(coefficient_count(B), dtype=np.complex128)
    u[omega_index(2, 1, 0)] = 1.0
    write("basis_B3_210.bin", ref.inverse(u, threads=1), manifest, B=3, what="reference ifsglft(unit omega(2,1,0))")
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print("wrote", len(manifest) - 3, "fixtures")


if __name__ == "__main__":
    main()
