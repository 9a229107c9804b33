"""The checked build (libraduls_gpu_checked.so, -DRG_CHECKED; csrc/common.cuh):
the race/bounds evidence on a GPU pool where compute-sanitizer does not run.

Every global record access of every kernel family (vector loads and stores,
TMA bulk copies, L2 prefetches, digit-array stores, peer stores) is checked
against the device ranges the call registered, TMA copies also for 16-B
alignment; mbarrier waits are bounded (a lost arrival is counted, not hung);
the scratch buffers and dynamic shared memory are poisoned with 0xA5 before
use (a read of anything not written first changes the output); and with
RADULS_GPU_CHECK_JITTER random __nanosleep at every producer/consumer
hand-off and named barrier perturbs warp interleavings, so an ordering race
turns into a parity failure. Any call that recorded a violation fails with
RADULS_GPU_EINTERNAL, so the parity suite run against the checked build
(compared byte for byte with the oracle) is the check. The reference argues
its own race freedom in prose (P/include/raduls/kernels.hpp:10-13, 157-159).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# the parity suite minus the 8-64 GiB full-size configs (minutes under the checks)
PARITY = ["tests/test_gpu_parity.py", "tests/test_gpu_kernels.py", "tests/test_gpu_lsd.py",
          "tests/test_gpu_local_edges.py", "tests/test_gpu_local_bitmap.py", "tests/test_gpu_fuzz.py", "tests/test_gpu_digit_array.py", "tests/test_gpu_progressive.py",
          "tests/test_gpu_distributed.py", "tests/test_gpu_multi.py"]
DESELECT = ("not full_size and not c5_full and not concurrent and not frees_its and not allocation_failure "
            "and not bench")


def _env(**kw):
    e = dict(os.environ, RADULS_GPU_LIB="checked")
    e.update(kw)
    return e


def _run(cmd, env, timeout=1800):
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_checked_library_reports_itself(torch_cuda):
    code = ("import numpy as np, ctypes as C, torch, paper_1612_02557_b200 as rg\n"
            "d = rg.generate(300000, rg.RecordLayout(16, 8), seed=3)\n"
            "rg.sort(d, 300000, rg.RecordLayout(16, 8)); torch.cuda.synchronize()\n"
            "assert rg.check_sorted(d, 300000, rg.RecordLayout(16, 8))[0] == 0\n"
            "r = np.zeros(6, dtype=np.uint64)\n"
            "k = rg._lib.load().raduls_gpu_check_report(r.ctypes.data_as(C.POINTER(C.c_uint64)))\n"
            "assert rg._lib.LIB_PATH.endswith('_checked.so') and k == 1, (k, rg._lib.LIB_PATH)\n"
            "assert r[0] == 0 and r[4] == 0 and r[5] > 0, r\n"
            "print('CHECKED OK', r.tolist())\n")
    res = _run([sys.executable, "-c", code], _env())
    assert res.returncode == 0 and "CHECKED OK" in res.stdout, res.stdout + res.stderr


def test_checked_library_catches_an_out_of_range_access(torch_cuda):
    """Negative control: every registered range 16 B short — the last record
    of the array falls outside — so a correct sort must be reported."""
    code = ("import paper_1612_02557_b200 as rg, torch\n"
            "d = rg.generate(300000, rg.RecordLayout(16, 8), seed=3)\n"
            "try:\n"
            "    rg.sort(d, 300000, rg.RecordLayout(16, 8)); torch.cuda.synchronize()\n"
            "except Exception as ex:\n"
            "    print('CAUGHT', type(ex).__name__, ex)\n")
    res = _run([sys.executable, "-c", code], _env(RADULS_GPU_CHECK_SHRINK="16"))
    assert "CAUGHT" in res.stdout, res.stdout + res.stderr
    assert "out-of-range" in res.stderr


def test_parity_suite_under_checked_build(torch_cuda):
    res = _run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-k", DESELECT, *PARITY], _env(),
               timeout=3000)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    import re
    m = re.search(r"(\d+) passed", res.stdout)
    assert m and int(m.group(1)) >= 150, res.stdout[-2000:]


def test_every_kernel_family_under_jitter(torch_cuda):
    """scripts/sanitize_driver.py (every kernel family on C1-C4-shaped inputs,
    both scatter ranking modes, the multi-GPU building blocks, checked against
    the oracle) with scheduling jitter, three times."""
    for mode in ("atomic", "ballot", "atomic"):
        env = _env(RADULS_GPU_CHECK_JITTER="1")
        if mode == "ballot":
            env["RADULS_GPU_STABLE_RANK"] = "ballot"
        res = _run([sys.executable, "scripts/sanitize_driver.py"], env)
        assert res.returncode == 0 and "DRIVER OK" in res.stdout, res.stdout[-3000:] + res.stderr[-3000:]
        assert "violations 0 timeouts 0" in res.stdout, res.stdout[-2000:]
