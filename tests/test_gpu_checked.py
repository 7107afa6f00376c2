"""Memory safety of the CUDA path without compute-sanitizer (closed on this GPU pool): the
checked build libbf_checked.so (build.py --checked, -DBF_CHECKED) bounds-checks every gathered
column index and the TMA tile copies, bounds the polling loops of the sync-free ILU sweeps,
checks the SpGEMM / transpose / renumbering writes, and validates every matrix a handle holds;
any failed check turns the public call into BF_ERR_CUDA "device check failed ...".  These tests
run the end-to-end drivers and a parity subset against that build in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, extra_env=None, timeout=900):
    env = dict(os.environ, BF_LIB="checked", **(extra_env or {}))
    return subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_checked_build_is_loaded_and_selftest_fires():
    code = ("import numpy as np, paper_1611_00127_b200 as bf\n"
            "from workload import make_system\n"
            "assert bf.LIB_PATH.endswith('libbf_checked.so'), bf.LIB_PATH\n"
            "prob, J, rhs = make_system(1, dims=(6, 5, 1))\n"
            "try:\n"
            "    bf.BFSolver(J.row_ptr, J.col_idx, J.vals.reshape(-1), prob.dims)\n"
            "    print('NO-ERROR')\n"
            "except bf.BFError as e:\n"
            "    print('ERR', e)\n")
    r = _run(["-c", code], {"BF_CHECK_SELFTEST": "1"})
    assert r.returncode == 0, r.stderr
    assert "device check failed in bf_api.cu" in r.stdout, r.stdout


def test_sanitize_case_under_checked_build():
    r = _run(["tools/sanitize_case.py"])
    assert r.returncode == 0 and "sanitize_case: OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


def test_parity_subset_under_checked_build():
    r = _run(["-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "tests/test_gpu_parity.py", "tests/test_gpu_cpr.py",
              "-k", "C1 or C3-20x17x15 or C4-40x9x16 or restart or boundary or hash_overflow or variants or options_parity"],
             timeout=1500)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
