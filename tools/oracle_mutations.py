#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r1 "What's weak" 1).

Copies oracle/, synth/ and tests/ to a scratch directory, applies ONE source mutation to
oracle/oracle.c (a plausible mistake: a dropped term, a wrong sign, a wrong constant), and
runs the CPU oracle tests there.  A pin set is adequate when every mutation turns at least
one test red.  Prints one JSON line per mutation and a summary; exit code 1 if any mutation
survives.

    python tools/oracle_mutations.py            # all mutations
    python tools/oracle_mutations.py cu1_drop   # one
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# name -> (passage it breaks, text to find in oracle.c, replacement)
MUTATIONS = {
    # R_{1:j-1,j} += C U1 (R-8, Alg. 8)
    "cu1_drop": ("R-8: R_{1:j-1,j} += C U1 deleted",
                 "  if (c0 > 0) orc_matmul(C, c0, U1, bj, c0, bj, bj, R + c0 * ldr, ldr, 0, 1);\n", ""),
    "cu1_overwrite": ("R-8: R_{1:j-1,j} = C U1 (accumulate flag dropped)",
                      "orc_matmul(C, c0, U1, bj, c0, bj, bj, R + c0 * ldr, ldr, 0, 1);",
                      "orc_matmul(C, c0, U1, bj, c0, bj, bj, R + c0 * ldr, ldr, 0, 0);"),
    "cu1_u2": ("R-8: C U2 instead of C U1",
               "orc_matmul(C, c0, U1, bj, c0, bj, bj, R + c0 * ldr, ldr, 0, 1);",
               "orc_matmul(C, c0, U2, bj, c0, bj, bj, R + c0 * ldr, ldr, 0, 1);"),
    "matmul_acc_ignored": ("orc_matmul accumulate mode ignored",
                           "      C[i + j * ldc] = accumulate ? C[i + j * ldc] + s : s;",
                           "      C[i + j * ldc] = s;"),
    "matmul_general_transposed": ("orc_matmul general mode reads B transposed",
                                  "        for (int64_t t = 0; t < r; ++t) s += A[i + t * lda] * B[t + j * ldb];",
                                  "        for (int64_t t = 0; t < r; ++t) s += A[i + t * lda] * B[j + t * ldb];"),
    # s = sqrt(m) u ||A||_F^2 (Alg. 4 l.2)
    "shift_sqrt_b": ("Alg. 4 l.2: sqrt(b) instead of sqrt(m)",
                     "    const double s = sqrt((double)m) * unit_roundoff * fro2;",
                     "    const double s = sqrt((double)b) * unit_roundoff * fro2;"),
    "shift_fro_not_squared": ("Alg. 4 l.2: ||A||_F instead of ||A||_F^2",
                              "    const double s = sqrt((double)m) * unit_roundoff * fro2;",
                              "    const double s = sqrt((double)m) * unit_roundoff * sqrt(fro2);"),
    "shift_u_eps": ("Alg. 4 l.2: u = 2^-52 (machine epsilon) instead of 2^-53",
                    "    const double s = sqrt((double)m) * unit_roundoff * fro2;",
                    "    const double s = sqrt((double)m) * 2.0 * unit_roundoff * fro2;"),
    "reorth_dropped": ("Alg. 8 l.7: re-orthogonalisation update skipped",
                       "    orc_sub_prod(Xj, ldx, X, ldx, C, c0, m, c0, bj);\n", ""),
}


def run(name: str, tests: str) -> dict:
    why, old, new = MUTATIONS[name]
    with tempfile.TemporaryDirectory(prefix="orcmut_") as d:
        for sub in ("oracle", "synth", "tests"):
            shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
        src = os.path.join(d, "oracle", "oracle.c")
        s = open(src).read()
        if s.count(old) != 1:
            return {"mutation": name, "error": f"pattern found {s.count(old)} times"}
        open(src, "w").write(s.replace(old, new))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu and not slow", tests,
                            "-p", "no:randomly"], cwd=d, capture_output=True, text=True)
        tail = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED") or " passed" in ln or " failed" in ln]
        return {"mutation": name, "breaks": why, "killed": r.returncode != 0, "pytest": tail[-2:]}


def main() -> int:
    names = sys.argv[1:] or list(MUTATIONS)
    res = [run(n, "tests/test_oracle.py") for n in names]
    for r in res:
        print(json.dumps(r))
    survivors = [r["mutation"] for r in res if not r.get("killed")]
    print(json.dumps({"mutations": len(res), "survivors": survivors}))
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
