"""The C++ drop-in headers (include/flashsvd_b200/) used as a reference-side
caller would: reference types, reference MemoryMeter, reference signatures.
tests/cpp/dropin_test.cpp compares each b200 call with the reference's own
CPU function (outputs within tolerance, identical meter event logs, same
exception types).  The binary is built in the build container by
__graft_entry__.build() (it links the reference objects from oracle/_ref)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_build", "dropin_test")


def _binary():
    if not os.path.exists(BIN):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
        else:
            pytest.skip("tests/cpp/_build/dropin_test not built (needs /root/reference at build time)")
    return BIN


def test_dropin_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "no CPU fallback" in r.stderr + r.stdout


@pytest.mark.gpu
def test_dropin_matches_reference_on_gpu():
    r = subprocess.run([_binary()], capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
