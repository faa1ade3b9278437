"""C-ABI boundary tests that need no GPU (-m "not gpu").

libcomet.so must load, export every entry point include/comet.h declares,
and reject bad arguments on the host before touching the device.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2410_12168_b200 import comet

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "comet.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(comet_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_paper_entry_points():
    fns = header_functions()
    for f in ("comet_quantize_act", "comet_pack_weight", "comet_w4ax_gemm"):
        assert f in fns
    assert set(fns) == set(comet.EXPORTS)


def test_library_loads_and_exports_every_header_symbol():
    L = comet.lib()
    for f in header_functions():
        assert hasattr(L, f), f
        assert ctypes.cast(getattr(L, f), ctypes.c_void_p).value


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {comet.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_sass_uses_tcgen05_and_tma():
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {comet.LIB_PATH} 2>/dev/null").read()
    assert "UTCIMMA" in sass or "UTCMMA" in sass  # tcgen05.mma kind::i8
    assert "UTMALDG" in sass                      # TMA tensor loads
    assert "LDTM" in sass                         # tcgen05.ld
    assert "HMMA" not in sass and "IMMA." not in sass.replace("UTCIMMA", "")


def test_size_helpers():
    L = comet.lib()
    bits = np.array([8, 4, 4, 8, 4], np.uint8)
    p = bits.ctypes.data_as(ctypes.c_void_p)
    assert L.comet_act_plane8_bytes(10, 640, p) == 10 * 256
    assert L.comet_act_plane4_bytes(10, 640, p) == 10 * 3 * 64
    assert L.comet_act_ldsx(10) == 12 and L.comet_act_ldsx(0) == 0 and L.comet_act_ldsx(-1) == -1
    assert L.comet_act_plane8_bytes(10, 600, p) == -1  # K % 128
    bad = np.array([8, 5], np.uint8)
    assert L.comet_act_plane8_bytes(1, 256, bad.ctypes.data_as(ctypes.c_void_p)) == -1
    assert L.comet_w4ax_gemm_workspace_bytes(16, 100, 512) == -1  # N % 128
    # prefill: the tile counters + the e4m3 token plane (M*K at most) + corrections (K/128 x ldsx fp32)
    assert L.comet_w4ax_gemm_workspace_bytes(4096, 4096, 4096) == 64 * 1024 + 4096 * 4096 + 32 * 4096 * 4
    assert L.comet_w4ax_gemm_workspace_bytes(16, 4096, 4096) > 64 * 1024  # decode: split-K partials


def _call_gemm(M=16, N=256, K=512, bits=(4, 4, 4, 8), group=128, ldsx=None, ldy=None, nulls=()):
    L = comet.lib()
    b = np.array(bits, np.uint8)
    fake = ctypes.c_void_p(1 << 20)  # never dereferenced: validation fails first
    g = lambda name: None if name in nulls else fake
    return L.comet_w4ax_gemm(g("Xq8"), g("Xq4"), g("Sx"), ldsx if ldsx is not None else M, b.ctypes.data_as(ctypes.c_void_p),
                             M, K, g("Wq"), g("Sw"), N, group, g("Y"), ldy if ldy is not None else N, None, 0, None)


@pytest.mark.parametrize("kw,status", [
    (dict(K=500, bits=(4, 4, 4, 4)), 2),         # K % 128
    (dict(N=200), 2),                            # N % 128
    (dict(group=64), 2),                         # group not in {128, K}
    (dict(bits=(4, 4, 4, 5)), 1),                # bad block_bits entry
    (dict(ldsx=15), 2),                          # ldsx < M
    (dict(ldsx=18), 2),                          # ldsx % 4
    (dict(M=-1), 1),
    (dict(ldy=128), 2),                          # ldy < N
    (dict(nulls=("Xq8",)), 1),                   # INT8 block present but no plane
    (dict(nulls=("Wq",)), 1),
])
def test_gemm_rejects_bad_arguments_before_launch(kw, status):
    assert _call_gemm(**kw) == status


def test_zero_sized_calls_are_noops():
    assert _call_gemm(M=0, ldsx=0) == 0
    assert _call_gemm(N=0) == 0


def test_quantize_rejects_bad_arguments():
    L = comet.lib()
    b = np.array([4, 8], np.uint8).ctypes.data_as(ctypes.c_void_p)
    fake = ctypes.c_void_p(1 << 20)
    q = lambda M=4, K=256, ldx=256, ldsx=4, X=fake, Xq8=fake, Xq4=fake, Sx=fake: L.comet_quantize_act(
        X, ldx, M, K, None, b, Xq8, Xq4, Sx, ldsx, None)
    assert q(K=200) == 2 and q(ldx=128) == 2 and q(ldx=260) == 2 and q(ldsx=3) == 2
    assert q(Xq8=None) == 1 and q(X=None) == 1
    assert q(X=ctypes.c_void_p((1 << 20) + 2)) == 3  # misaligned
    assert q(M=0, ldsx=0) == 0


def test_pack_weight_rejects_bad_arguments():
    L = comet.lib()
    fake = ctypes.c_void_p(1 << 20)
    p = lambda N=128, K=256, group=128, ldw=256: L.comet_pack_weight(fake, ldw, N, K, None, group, fake, fake, None)
    assert p(group=64) == 2 and p(K=100) == 2 and p(ldw=200) == 2 and p(N=-1) == 1 and p(N=0) == 0


def test_status_strings():
    L = comet.lib()
    for k, v in comet.STATUS.items():
        assert L.comet_status_str(k).decode() == v


def test_product_path_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2410_12168_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "comet_oracle" not in src, f
