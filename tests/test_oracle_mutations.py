"""Mutation check of the oracle's pins (VERDICT r1 "weak 1"): every pin must bite.

Each case plants one plausible mistake in a copy of oracle/oracle.c -- a dropped term, a flipped
sign, a missing filter -- builds it, and runs the oracle pin suite (tests/test_oracle.py,
tests/test_oracle_cpr.py) against that build through ORACLE_SO.  The suite must FAIL for every
mutant.  A case whose source line is not found fails too, so the list follows the oracle's code.
"""
import concurrent.futures as cf
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")

# (name, exact source text, replacement, count of occurrences to replace (0 = all))
MUTANTS = [
    # classical interpolation (Q26 / R6 / R8)
    ("strong-F distribution weight c = a_ik/D_k set to 0", "double c = aik / Dk;", "double c = 0.0 * (aik / Dk);", 1),
    ("strong-F distribution weight scaled by 0.8", "double c = aik / Dk;", "double c = 0.8 * (aik / Dk);", 1),
    ("weak connections not lumped into the diagonal", "else if (!strong[q]) dg = dg + A->v[q];",
     "else if (!strong[q]) dg = dg;", 1),
    ("no common C point: a_ik not lumped into the diagonal", "dg = dg + aik;", "dg = dg;", 1),
    ("sign filter a-bar dropped", "double abar = (sk * A->v[t] < 0.0) ? A->v[t] : 0.0;", "double abar = A->v[t];", 0),
    ("diagonal sign of row i used for the strong F neighbour k", "double sk = diag_sign(A, k);",
     "double sk = diag_sign(A, i);", 1),
    # GMRES with CGS2 (Q30)
    ("CGS2 correction h += h' dropped", "for (int32_t i = 0; i <= j; i++) h[i] += h2[i];", "", 1),
    ("Givens rotation sign flipped in g", "g[j + 1] = -sn[j] * g[j];", "g[j + 1] = sn[j] * g[j];", 1),
    ("second CGS pass projects with h instead of h'", "w[t] -= h2[i] * V[(size_t)i * N + t];",
     "w[t] -= h[i] * V[(size_t)i * N + t];", 1),
    # S~, strength (Q24), smoother (Q27), Galerkin (c.2 3.5), PMIS (Q25)
    ("S~ update sign flipped", "S->v[p] = S->v[p] - prod;", "S->v[p] = S->v[p] + prod;", 1),
    ("strength: sign of the diagonal ignored", "strong[q] = (uint8_t)(m > 0.0 && A->ci[q] != i && -sg * A->v[q] >= thr);",
     "strong[q] = (uint8_t)(m > 0.0 && A->ci[q] != i && -A->v[q] >= thr);", 1),
    ("l1 diagonal without absolute values", "s = s + fabs(A->v[q]);", "s = s + A->v[q];", 1),
    ("Chebyshev interval ignores the estimated upper end hi (R21)",
     "double theta = hi * (1.0 + lo) / 2.0, delta = hi * (1.0 - lo) / 2.0;",
     "double theta = (1.0 + lo) / 2.0, delta = (1.0 - lo) / 2.0;", 1),
    ("power estimate without the D^-1 scaling", "w[i] = w[i] / d[i];", "w[i] = w[i];", 1),
    ("Chebyshev recurrence coefficient 2 rho_new / delta halved",
     "dir[i] = rho_new * rho * dir[i] + (2.0 * rho_new / delta) * ((b[i] - tmp[i]) / d[i]);",
     "dir[i] = rho_new * rho * dir[i] + (rho_new / delta) * ((b[i] - tmp[i]) / d[i]);", 1),
    ("Galerkin product drops the last term of each row", "acc[J] = acc[J] + prod;",
     "if (t + 1 < B->rp[k + 1] || q + 1 < A->rp[i + 1]) acc[J] = acc[J] + prod;", 1),
    ("PMIS index tie-break reversed", "(key[a] == key[b] && (a) > (b))", "(key[a] == key[b] && (a) < (b))", 1),
    ("V-cycle post-smoother skipped", "for (int s = 0; s < h->opt.nu_post; s++) smooth(h, l, b, x, tmp, dir);", "", 1),
    ("BF apply: A_ps coupling sign flipped", "rp[c] = rp[c] - t[c];", "rp[c] = rp[c] + t[c];", 1),
    ("R23 stop at a non-positive Galerkin diagonal accepts a zero diagonal", "if (!(aii > 0.0)) return 0;",
     "if (aii < -1e300) return 0;", 1),
    ("block ILU(0): fill update sign flipped", "lu[4 * t + e] = lu[4 * t + e] - P[e];", "lu[4 * t + e] = lu[4 * t + e] + P[e];", 1),
]


def _mutate(src, old, new, count):
    n = src.count(old)
    if n == 0 or (count and n != count):
        raise AssertionError(f"mutation anchor found {n} times (want {count or '>= 1'}): {old!r}")
    return src.replace(old, new)


def _run_mutant(args):
    name, old, new, count, tmp = args
    src = open(SRC).read()
    mutated = _mutate(src, old, new, count)
    tag = "".join(ch if ch.isalnum() else "_" for ch in name)[:60]
    c = os.path.join(tmp, tag + ".c")
    so = os.path.join(tmp, tag + ".so")
    with open(c, "w") as f:
        f.write(mutated)
    import oracle
    subprocess.check_call(["gcc", *oracle.CFLAGS, "-I", os.path.join(ROOT, "oracle"), c, "-o", so, "-lm"])
    env = dict(os.environ, ORACLE_SO=so)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "not gpu",
                        os.path.join(ROOT, "tests", "test_oracle.py"), os.path.join(ROOT, "tests", "test_oracle_cpr.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    last = [l for l in r.stdout.splitlines() if l.strip()][-1:] or [""]
    return name, r.returncode, last[0]


def test_every_mutant_fails_a_pin():
    with tempfile.TemporaryDirectory() as tmp:
        jobs = [(name, old, new, count, tmp) for name, old, new, count in MUTANTS]
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
            results = list(ex.map(_run_mutant, jobs))
    survivors = [(name, last) for name, rc, last in results if rc == 0]
    errors = [(name, rc, last) for name, rc, last in results if rc not in (0, 1)]
    assert not errors, errors
    assert not survivors, f"mutants not caught by any pin: {survivors}"


def test_unmutated_oracle_passes_through_oracle_so():
    """The harness itself: the unmodified source built the same way passes the pin suite."""
    with tempfile.TemporaryDirectory() as tmp:
        name, rc, last = _run_mutant(("unmodified", "#include <math.h>", "#include <math.h>", 1, tmp))
    assert rc == 0, last
