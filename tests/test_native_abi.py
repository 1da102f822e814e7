"""The C ABI library loads and exports every entry point include/blp.h declares.

No compute call is made (no GPU here): only the symbol table and the pure host
helpers (ABI version, shape support, kernel-variant selection).
"""
import ctypes
import re
from pathlib import Path

import pytest

from paper_1802_08557_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "blp.h"


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(blp_\w+)\s*\(", text)))


def test_header_declares_the_exported_set():
    assert declared_functions() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [name for name in declared_functions() if not hasattr(lib, name)]
    assert not missing, f"libblp.so lacks {missing}"


def test_host_only_entry_points():
    lib = _native.load()
    assert lib.blp_abi_version() == 1
    assert lib.blp_shape_supported(28, 32) == 1
    assert lib.blp_shape_supported(-1, 3) == 0
    assert lib.blp_last_error() == b""
    assert lib.blp_launch_count() >= 0


@pytest.mark.parametrize("m,n,family", [(5, 5, "ctab_r1_s8"), (28, 32, "ctab_r1_s32"), (64, 32, "lazy+cm2_r16_s16"),
                                        (100, 100, "lazy+cm4_r48_s56"), (50, 50, "lazy+cm2_r64_s0"), (100, 150, "lazy+smem"),
                                        (90, 140, "lazy+smem"), (64, 40, "lazy+cm2_r64_s0"),
                                        (500, 500, "lazy+cluster"),
                                        (150, 150, "lazy+cm8_r96_s104"), (300, 150, "lazy+cluster"), (600, 600, "lazy+hbm")])
def test_kernel_variant_selection(m, n, family):
    assert _native.kernel_variant(m, n).startswith(family)


@pytest.mark.parametrize("m,n,family", [(64, 8, "ctab_r2_s8"), (128, 8, "ctab_r4_s8"), (64, 16, "ctab_r2_s16"),
                                        (40, 16, "lazy+cm2_r16_s16"), (100, 16, "lazy+cm4_r32_s0"),
                                        (200, 8, "lazy+cm8")])
def test_narrow_lps_dispatch(m, n, family, monkeypatch):
    """Narrow LPs (n <= 8, or n <= 16 at 49..64 rows) go to the one-warp condensed kernel
    (measured faster than the multi-warp form plus its lazy pre-pass); BLP_CMULTI=3 forces
    the multi-warp form for every 33..128-row shape; beyond 128 rows there is no one-warp form."""
    assert _native.kernel_variant(m, n) == family or _native.kernel_variant(m, n).startswith(family)
    monkeypatch.setenv("BLP_CMULTI", "3")
    v = _native.kernel_variant(m, n)
    assert v.startswith("lazy+cm"), v


def test_kernel_variant_support_mode():
    """Support mode (one A, b): the condensed kernels run without the lazy pass ahead of
    them (their shared phase 1 applies instead)."""
    assert _native.kernel_variant(64, 32, True) == "cm2_r16_s16"
    assert _native.kernel_variant(28, 32, True) == "ctab_r1_s32"
    assert _native.kernel_variant(100, 100, True) == "cm4_r48_s56"


def test_invalid_arguments_rejected_without_cuda():
    lib = _native.load()
    lim = _native.make_limits()
    rc = lib.blp_solve_batch_host(None, None, None, -1, 2, 2, 0, ctypes.byref(lim), None, None, None, None,
                                  None, 0)
    assert rc == -1 and b"invalid" in lib.blp_last_error()
