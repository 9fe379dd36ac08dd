#!/usr/bin/env python
"""Mutation check of the oracle's pins.

Each mutant is one plausible mistake written into oracle/fdgs_oracle.c (a
dropped term, a wrong sign, index or operand order, a removed clamp); it is
compiled to /tmp and the -m "not gpu" oracle pin suites are run against it
(ORACLE_LIB).  Every mutant must make at least one pin fail ("killed").

    python tools/mutate_oracle.py [--json profiles/r02_oracle_mutants.json]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "fdgs_oracle.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_projection_pins.py", "tests/test_oracle_stv.py"]

# (name, exact text in fdgs_oracle.c, replacement)
MUTANTS = [
    ("dilation dropped", "a2 = a2 + OR_DIL;", "a2 = a2;"),
    ("sign in L(q)", "{b, a, -d, c}", "{b, a, d, c}"),
    ("R(q) row swapped", "{q, p, s, -r}, {r, -s, p, q}", "{r, -s, p, q}, {q, p, s, -r}"),
    ("depth tie by descending index", "return (x->idx > y->idx) - (x->idx < y->idx);",
     "return (x->idx < y->idx) - (x->idx > y->idx);"),
    ("Schur term dropped", "Nm[k][j] = fma(-v[k], M[3][j], M[k][j]);", "Nm[k][j] = M[k][j];"),
    ("sign of dt", "const double dt = t - (double)mu[3];", "const double dt = (double)mu[3] - t;"),
    ("SH constant (Y6)", "Y[6] = k2b * (2.0 * zz - xx - yy);", "Y[6] = k2b * (2.0 * zz - xx + yy);"),
    ("SH sign (Y1)", "Y[1] = -k1 * y;", "Y[1] = k1 * y;"),
    ("SH sign (Y13)", "Y[13] = -k3c * x * (4.0 * zz - xx - yy);", "Y[13] = k3c * x * (4.0 * zz - xx - yy);"),
    ("termination threshold", "const int stop = test < OR_T_STOP;", "const int stop = test < 1e-3;"),
    ("temporal threshold", "const double kts = OR_KT * s44;", "const double kts = 0.9 * OR_KT * s44;"),
    ("transposed camera rotation", "Rc[r][c] = (double)cam->R[r * 3 + c];", "Rc[r][c] = (double)cam->R[c * 3 + r];"),
    ("sign of j02", "const double j02 = -((fx * cxz) * rz)", "const double j02 = ((fx * cxz) * rz)"),
    ("sign of j12", "j12 = -((fy * cyz) * rz);", "j12 = ((fy * cyz) * rz);"),
    ("Jacobian clamp removed (x)", "const double cxz = fmin(fmax(xz, -limx), limx);", "const double cxz = xz;"),
    ("Jacobian clamp removed (y)", "const double cyz = fmin(fmax(yz, -limy), limy);", "const double cyz = yz;"),
    ("Jacobian clamp 1.0 x half-FOV", "#define OR_JCLAMP  1.3", "#define OR_JCLAMP  1.0"),
    ("view direction reversed", "for (int k = 0; k < 3; ++k) d[k] = g->mu3[k] - ccam[k];",
     "for (int k = 0; k < 3; ++k) d[k] = ccam[k] - g->mu3[k];"),
    ("camera centre = -T", "ccam[k] = -(Rc[0][k] * Tc[0] + Rc[1][k] * Tc[1] + Rc[2][k] * Tc[2]);",
     "ccam[k] = -Tc[k];"),
    ("alpha clamp removed", "if (alpha > OR_ALPHA_MAX) alpha = OR_ALPHA_MAX;", ""),
    ("AABB shrunk", "const double hx = fma(sqrt(q2 * a2), OR_MARGIN_MUL, OR_MARGIN_ADD);",
     "const double hx = 0.9 * sqrt(q2 * a2);"),
    ("conic B sign", "B = -(b2 * rdet)", "B = (b2 * rdet)"),
    ("mask OR -> AND", "out[w] = a[w] | b[w];", "out[w] = a[w] & b[w];"),
    ("bracket: right key-frame off by one", "for (int k = nk - 1; k >= 0; --k) if (kf[k] >= frame) ri = k;",
     "for (int k = nk - 1; k >= 0; --k) if (kf[k] > frame) ri = k;"),
    ("j00 from fy", "const double j00 = fx * rz, j11 = fy * rz;", "const double j00 = fy * rz, j11 = fy * rz;"),
    ("Jacobian y clamp from the width", "const double limy = OR_JCLAMP * ((double)cam->height / (2.0 * fy));",
     "const double limy = OR_JCLAMP * ((double)cam->width / (2.0 * fy));"),
    ("u from cy", "const double u = fma(fx, xz, cx), vv = fma(fy, yz, cy);",
     "const double u = fma(fx, xz, cy), vv = fma(fy, yz, cy);"),
    ("S^TV uses p instead of p2", "return 1.0 / (0.5 * tanh(fabs(p2)) + 0.5);", "return 1.0 / (0.5 * tanh(fabs(p)) + 0.5);"),
]


def run(mutant, tmp):
    name, old, new = mutant
    src = open(SRC).read()
    if src.count(old) != 1:
        return dict(name=name, status="not-applicable", detail=f"text found {src.count(old)} times")
    path_c = os.path.join(tmp, "mut.c")
    path_so = os.path.join(tmp, f"mut_{abs(hash(name))}.so")
    with open(path_c, "w") as fh:
        fh.write(src.replace(old, new))
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                           "-fno-fast-math", "-o", path_so, path_c, "-lm"])
    env = dict(os.environ, ORACLE_LIB=path_so, PYTHONPATH=ROOT)
    t0 = time.time()
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *PINS], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=1200)
    failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED ")]
    return dict(name=name, status="killed" if r.returncode != 0 else "SURVIVED", killed_by=failed[:1],
                seconds=round(time.time() - t0, 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    res = []
    with tempfile.TemporaryDirectory() as tmp:
        for m in MUTANTS:
            out = run(m, tmp)
            print(json.dumps(out), flush=True)
            res.append(out)
    survived = [r["name"] for r in res if r["status"] != "killed"]
    summary = dict(mutants=len(res), killed=sum(r["status"] == "killed" for r in res), not_killed=survived,
                   suites=PINS, results=res)
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(summary, fh, indent=1)
    print(json.dumps({k: summary[k] for k in ("mutants", "killed", "not_killed")}))
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
