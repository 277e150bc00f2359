"""Implementation variants chosen by the plan (or forced by environment
switches, read once per process, hence subprocesses) must agree:

* R row maxima by the lattice DP vs the direct gather pass: same maxima, so the
  same R slices and a bit-identical backward;
* V^T slices from the forward's aux warps vs the all-SM pack kernel: same bytes,
  bit-identical backward inside the descent;
* next-step V^T slices from the backward's update vs packed by the forward,
  and the fused update vs the split one (gradient stored, all-SM k_update):
  the descent agrees to the slice precision;
* narrow tiles vs full 160-wide grid tiles: the same integer products, so a
  bit-identical plain backward; the descent (forward atomics in another order)
  agrees to fp32 rounding.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPE = ("9", "4", "700")  # N = 495: several tiles, a narrow last column block (700 = 4*160 + 60)


def _run(tmp_path, tag, env):
    out = str(tmp_path / f"{tag}.npz")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "variant_grad.py"), *SHAPE, out], env=e,
                   check=True, timeout=300)
    return np.load(out)


@pytest.mark.gpu
def test_rmax_dp_vs_direct(tmp_path):
    a = _run(tmp_path, "dp", {"SOS_RPACK_TWOPASS": "0"})
    b = _run(tmp_path, "direct", {"SOS_RPACK_TWOPASS": "1"})
    assert np.array_equal(a["grad"], b["grad"])


@pytest.mark.gpu
def test_vtq_aux_vs_kernel(tmp_path):
    a = _run(tmp_path, "aux", {"SOS_VTQ_AUX": "1"})
    b = _run(tmp_path, "kernel", {"SOS_VTQ_AUX": "0"})
    assert np.array_equal(a["grad"], b["grad"])
    rel = np.linalg.norm(a["V3"] - b["V3"]) / np.linalg.norm(a["V3"])
    assert rel <= 1e-6
    assert np.allclose(a["losses"], b["losses"], rtol=1e-5)


@pytest.mark.gpu
def test_narrow_vs_full_tiles(tmp_path):
    a = _run(tmp_path, "narrow", {"SOS_NARROW_TILES": "1"})
    b = _run(tmp_path, "full", {"SOS_NARROW_TILES": "0"})
    assert np.array_equal(a["grad"], b["grad"])
    rel = np.linalg.norm(a["V3"] - b["V3"]) / np.linalg.norm(a["V3"])
    assert rel <= 1e-6
    assert np.allclose(a["losses"], b["losses"], rtol=1e-5)


@pytest.mark.gpu
def test_vtq_from_update_vs_forward_pack(tmp_path):
    a = _run(tmp_path, "upd", {"SOS_VTQ_UPDATE": "1", "SOS_UPDATE_SPLIT": "0"})
    b = _run(tmp_path, "fwd", {"SOS_VTQ_UPDATE": "0", "SOS_UPDATE_SPLIT": "0"})
    assert np.array_equal(a["grad"], b["grad"])  # sos_backward does not use it
    rel = np.linalg.norm(a["V3"] - b["V3"]) / np.linalg.norm(a["V3"])
    assert rel <= 1e-6
    assert np.allclose(a["losses"], b["losses"], rtol=1e-5)


@pytest.mark.gpu
def test_update_fused_vs_split(tmp_path):
    a = _run(tmp_path, "fused", {"SOS_UPDATE_SPLIT": "0"})
    b = _run(tmp_path, "split", {"SOS_UPDATE_SPLIT": "1"})
    assert np.array_equal(a["grad"], b["grad"])
    rel = np.linalg.norm(a["V3"] - b["V3"]) / np.linalg.norm(a["V3"])
    assert rel <= 1e-6
    assert np.allclose(a["losses"], b["losses"], rtol=1e-5)
