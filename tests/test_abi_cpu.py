# SPDX-License-Identifier: Apache-2.0
"""CPU: the C-ABI library loads, exports every symbol include/staleflow/train_math.h
declares, keeps the struct layout the header defines, maps errors onto
staleflow::Errc without crashing, and the product path has no CPU fallback."""
import ctypes
import os
import subprocess
import textwrap

import pytest

from paper_2604_11554_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_function():
    names = _lib.header_functions()
    assert len(names) >= 17
    l = _lib.lib()
    missing = [n for n in names if not hasattr(l, n)]
    assert not missing, missing
    # and every binding in _lib refers to a declared function
    assert set(_lib._SIGS) <= set(names)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = {ln.split(".")[-2] for ln in out.splitlines() if ln.strip().endswith(".cubin")}
    assert archs == {"sm_100a"}, out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    # Blackwell-native evidence: TMA bulk copies, tcgen05 TMEM stores/loads, packed fp32x2 math
    for op in ("UBLKCP", "STTM", "LDTM", "FFMA2", "MUFU.EX2"):
        assert op in sass, op


def test_abi_version_and_defaults():
    l = _lib.lib()
    assert l.sf_tm_abi_version() == 1
    p = _lib.default_loss_params()
    assert abs(p.clip_eps_low - 0.2) < 1e-7 and abs(p.clip_eps_high - 0.28) < 1e-7
    assert p.dual_clip_c == 0 and p.kl_beta == 0 and p.entropy_coef == 0 and p.inv_temperature == 1
    assert p.norm_mode == _lib.NORM_TOKEN_MEAN and p.masked_rows == _lib.MASKED_ZERO_FILL


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(textwrap.dedent("""
        #include <stdio.h>
        #include <stddef.h>
        #include "staleflow/train_math.h"
        int main(void) {
          printf("%zu %zu %zu %zu %zu\\n", sizeof(sf_tm_loss_params), offsetof(sf_tm_loss_params, norm_mode),
                 offsetof(sf_tm_loss_params, inv_norm), offsetof(sf_tm_loss_params, masked_rows),
                 (size_t)SF_TM_NUM_METRICS);
          return 0;
        }"""))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    P = _lib.LossParams
    assert vals == [ctypes.sizeof(P), P.norm_mode.offset, P.inv_norm.offset, P.masked_rows.offset, _lib.NUM_METRICS]


def test_errors_map_to_errc_without_crashing():
    l = _lib.lib()
    assert l.sf_tm_last_error(None) == b"null handle"
    assert l.sf_tm_destroy(None) == _lib.OK
    null = None
    # every entry point refuses a NULL handle with ConfigError (21)
    assert l.sf_tm_logprob_fwd(null, None, 0, 0, 1, 1, None, 1.0, None, None, None, None) == _lib.CONFIG_ERROR
    assert l.sf_tm_grpo_advantage(null, None, None, 0, 1e-6, 0, None, None, None) == _lib.CONFIG_ERROR
    assert l.sf_tm_pg_loss_fwd_bwd(null, None, 0, 0, 1, 1, None, None, None, None, None, None, None, 1,
                                   None, None, None, None) == _lib.CONFIG_ERROR
    assert l.sf_tm_create(0, None) == _lib.CONFIG_ERROR


def test_create_without_gpu_is_internal():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = _lib._H()
    assert _lib.lib().sf_tm_create(0, ctypes.byref(h)) == _lib.INTERNAL


def test_product_path_has_no_cpu_fallback(monkeypatch):
    import torch

    from paper_2604_11554_b200 import train_math as tm

    with pytest.raises(_lib.TrainMathError) as e:
        tm.logprob_fwd(torch.zeros(2, 8), torch.zeros(2, dtype=torch.int32))
    assert e.value.code == _lib.CONFIG_ERROR
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libsf_train_math.so")
    with pytest.raises(ImportError):
        _lib.lib()


def test_product_package_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_2604_11554_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".hpp")) or f == "Makefile":
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", '#include "sf_oracle', "libsf_oracle", "oracle/_build"):
                    assert bad not in txt, (f, bad)


def test_seam_library_exports_every_header_function():
    """libsf_seam.so (the C++ trainer seam behind a C-ABI) exports every
    function include/staleflow/train_math_seam_c.h declares; a batch encodes
    without a GPU."""
    import numpy as np

    from paper_2604_11554_b200 import seam

    names = seam.header_functions()
    l = seam.lib()
    assert names and not [n for n in names if not hasattr(l, n)]
    assert set(seam._SIGS) <= set(names)
    b = seam.MicroBatch([3, 2], np.arange(5), np.zeros(5), np.zeros(5), [0.5, -0.5], True,
                        loss_mask=np.ones(5, np.uint8))
    assert b.T == 5 and b.B == 2
    import torch

    if not torch.cuda.is_available():  # no device: the seam reports Internal, it does not crash
        s = ctypes.c_void_p()
        assert l.sf_seam_create(0, ctypes.byref(s)) == _lib.INTERNAL
