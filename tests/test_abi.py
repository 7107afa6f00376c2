"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports every
symbol include/bf.h declares (no compute call needs a GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bf.h")).read()
    return sorted(set(re.findall(r"^(?:bf_status|const char \*|int64_t)\s*(bf_\w+)\s*\(", src, re.M)))


def _build():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bf_build", os.path.join(ROOT, "paper_1611_00127_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


def test_library_builds_and_exports():
    so = _build()
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bf_\w+)", out))
    decl = declared_symbols()
    assert len(decl) >= 14
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    from paper_1611_00127_b200 import binding
    assert sorted(binding.EXPORTS) == decl


def test_sm100a_code_and_no_oracle_link():
    so = _build()
    out = subprocess.run(["cuobjdump", "-lelf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
    assert "oracle" not in deps
    # the product path never imports, includes or loads the oracle
    pkg = os.path.join(ROOT, "paper_1611_00127_b200")
    bad = re.compile(r"(^\s*(import|from)\s+oracle\b)|liboracle|oracle\.h|oracle/|import_module\(.oracle", re.M)
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                assert not bad.search(open(os.path.join(dp, f)).read()), f


def test_default_options_without_gpu():
    from paper_1611_00127_b200 import bf_default_options
    o = bf_default_options()
    assert o.theta == 0.25 and o.max_coarse == 64 and o.nu_pre == 1 and o.interp_norm == 1
    assert o.precond == 0  # BF (Algorithm 3); 1, 2 CPR-AMG(1)/(2), 3 coupled AMG
    # R22: Chebyshev(2) on [0.1, 1] for A_ss, l1-Jacobi for S~ (and A_pp, J); the oracle agrees
    assert (o.smoother, o.smoother_p, o.cheb_degree, o.cheb_lo, o.cheb_levels, o.cheb_eig) == (1, 0, 2, 0.1, 0, 0)
    assert o.diag_stop == 1  # R23
    import oracle
    oo = oracle.default_options()
    for f, _ in oracle.Options._fields_:
        assert getattr(oo, f) == getattr(o, f), f
    # the binding's struct mirrors include/bf.h field by field (a missing field would shift the rest)
    import ctypes
    from paper_1611_00127_b200 import binding
    src = open(os.path.join(ROOT, "include", "bf.h")).read()
    body = src[src.index("typedef struct {\n  double theta;"):src.index("} bf_options;")]
    decls = re.findall(r"^\s*(?:double|int32_t|uint64_t)\s+([\w\s,]+);", body, re.M)
    fields = [f.strip() for d in decls for f in d.split(",")]
    assert [f for f, _ in binding.bf_options._fields_] == fields


def test_oracle_struct_mirrors():
    """oracle/__init__.py's ctypes mirrors of or_options and or_bf follow oracle.h field by field."""
    import oracle
    src = open(os.path.join(ROOT, "oracle", "oracle.h")).read()

    def fields(tag):
        body = src[src.rindex("typedef struct {", 0, src.index("} " + tag + ";")):src.index("} " + tag + ";")]
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        out = []
        types = r"(?:double|int32_t|uint64_t|int64_t|int8_t|uint8_t|or_csr|or_amg|or_options)"
        for stmt in body.split(";"):
            m = re.match(r"\s*" + types + r"\s+(.+)$", stmt.replace("typedef struct {", ""), re.S)
            if not m:
                continue
            for f in m.group(1).split(","):
                out.append(re.sub(r"[\*\s]|\[.*\]", "", f))
        return out

    assert [f for f, _ in oracle.Options._fields_] == fields("or_options")
    names = [f for f, _ in oracle.BFs._fields_]
    want = fields("or_bf")
    assert names == want, (names, want)
