"""The reference's own doctest suite (proj/tests/*.cpp, 72 cases) compiled
unchanged against (a) the reference library -- validates the oracle build --
and (b) this repo's drop-in library.  On a CPU-only host the 16 cases that
reach the GPU hot path must fail loudly (no CPU fallback); on a B200 all 72
must pass (tests/test_gpu_api.py)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")
B200_TESTS = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests_b200")


def run(exe):
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", p.stdout)
    assert m, p.stdout + p.stderr
    return int(m.group(1)), int(m.group(2)), int(m.group(3)), p


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="oracle/_ref not built")
def test_reference_suite_passes_on_reference_library():
    total, passed, failed, _ = run(REF_TESTS)
    assert (total, passed, failed) == (72, 72, 0)


@pytest.mark.skipif(not os.path.exists(B200_TESTS), reason="oracle/_ref not built")
@pytest.mark.skipif(_has_gpu(), reason="CPU-only expectation")
def test_reference_suite_against_b200_library_without_gpu():
    total, passed, failed, p = run(B200_TESTS)
    assert total == 72
    # every failure is the loud no-device error, never a wrong answer
    errors = [l for l in p.stderr.splitlines() if "FAILED" in l or "threw" in l]
    assert failed == len(errors) and failed > 0
    assert all("no CPU fallback" in l for l in errors), "\n".join(errors)
    assert passed == 72 - failed
