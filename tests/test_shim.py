"""The C++ drop-in (include/lumi/cuda_renderer.h) exercised from the reference's side by the
compiled test binary tests/cpp/build/test_shim (reference template vs B200 overload)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, load_occ

BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_shim")


@pytest.mark.gpu
def test_reference_call_site_renders_on_b200(tmp_path):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/build/test_shim missing: build() compiles it where the "
                    "reference checkout exists")
    bits, res, _ = load_occ("small-T19")
    raw = tmp_path / "occ.raw"
    bits.astype(np.uint8).tofile(raw)
    r = subprocess.run([BIN, str(raw)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "OK" in r.stdout


@pytest.mark.gpu
def test_reference_training_loop_backward_on_b200(tmp_path):
    """include/lumi/cuda_train.h vs the reference's per-ray training loop (trainer.cpp:549-562)
    compiled from its own templates: loss terms rel 1e-6, gradients 1e-4 of max."""
    binp = os.path.join(ROOT, "tests", "cpp", "build", "test_train_shim")
    if not os.path.exists(binp):
        pytest.fail("tests/cpp/build/test_train_shim missing: build() compiles it where the "
                    "reference checkout exists")
    bits, res, _ = load_occ("small-T19")
    raw = tmp_path / "occ.raw"
    bits.astype(np.uint8).tofile(raw)
    r = subprocess.run([binp, str(raw)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "OK" in r.stdout
