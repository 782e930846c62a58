# SPDX-License-Identifier: Apache-2.0
"""The seams driven by the reference's own data plane:
TransferQueue / StreamLoader / StalenessGate compiled from /root/reference by
`make -C oracle bus` (test infrastructure, prebuilt into oracle/_ref so the GPU
box needs no reference tree), the product seams of
include/staleflow/train_math_seam.hpp on top (tests/cpp/test_bus_seam.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def _binary(name):
    exe = os.path.join(REF, name)
    if not os.path.exists(exe) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "bus"], check=True)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs the reference tree once: make -C oracle bus)")
    return exe


def test_bus_group_assembly_version_boundaries_staleness_cpu():
    out = subprocess.run([_binary("test_bus_seam_cpu"), "cpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "BUS CPU OK" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
def test_bus_driven_seams_gpu():
    """ActorLossSeam::step on bus-delivered micro-batches == the C-ABI on the same
    arrays (bitwise); version-boundary normalisation == the explicit-N run; the
    R3 record uploaded token-major and transposed on device == the host codec
    (FNV digest); Advantages over complete groups only."""
    out = subprocess.run([_binary("test_bus_seam_gpu"), "gpu"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "BUS GPU OK" in out.stdout, out.stdout + out.stderr
