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
