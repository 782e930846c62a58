# SPDX-License-Identifier: Apache-2.0
"""The C++ trainer-seam adapter (include/staleflow/train_math_seam.hpp):
MicroBatch payload codec on CPU (also compiled against the reference's own
staleflow::MicroBatch when /root/reference is present), and on a B200 the
adapter's step == the C-ABI seam call, bitwise."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_seam.cpp")
LIBDIR = os.path.join(ROOT, "paper_2604_11554_b200", "lib")
REF_INC = "/root/reference/proj/include"


def _build(tmp_path, name, extra, libs=(), compiler="g++"):
    exe = str(tmp_path / name)
    cmd = [compiler, "-Wall", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), *extra, SRC, "-o", exe,
           "-L", LIBDIR, "-lsf_train_math", f"-Wl,-rpath,{LIBDIR}", *libs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return exe


def test_seam_codec_cpu(tmp_path):
    exe = _build(tmp_path, "seam_mirror", [])
    out = subprocess.run([exe, "pack"], capture_output=True, text=True)
    assert out.returncode == 0 and "PACK OK" in out.stdout, out.stdout + out.stderr


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference tree not present (GPU box)")
def test_seam_codec_against_reference_microbatch(tmp_path):
    exe = _build(tmp_path, "seam_ref", ["-DSF_USE_REF_TYPES", "-I", REF_INC])
    out = subprocess.run([exe, "pack"], capture_output=True, text=True)
    assert out.returncode == 0 and "PACK OK" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
def test_seam_step_matches_c_abi(tmp_path):
    cuda = "/usr/local/cuda"
    exe = _build(tmp_path, "seam_gpu", ["-DSF_WITH_CUDA", "-I", f"{cuda}/include"],
                 libs=["-L", f"{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{cuda}/lib64"])
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "GPU OK" in out.stdout, out.stdout + out.stderr
