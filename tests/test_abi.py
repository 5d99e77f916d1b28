"""The C-ABI boundary (include/preft.h) without a GPU: the library loads,
exports every declared symbol, the ctypes mirror matches the C layout, status
codes map to the reference's exception classes, and the product path refuses
to run without CUDA (no silent CPU fallback)."""

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2605_14217_b200 import _lib, errors

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "preft.h"


def declared_functions() -> set[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    text = re.sub(r"#define.*", "", text)
    return set(re.findall(r"\b(preft_\w+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()  # raises if libpreft.so is missing
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), f"libpreft.so does not export {name}"
        assert name in _lib.SIGNATURES, f"no ctypes signature for {name}"
    assert set(_lib.SIGNATURES) == names


def test_host_only_entry_points():
    lib = _lib.load()
    assert lib.preft_abi_version() == _lib.ABI_VERSION
    assert lib.preft_meta_entries_words(10) == 2 + 3 * 10 + 1
    assert lib.preft_status_string(1) == b"ShapeError"
    assert lib.preft_status_string(7) == b"SyncError"


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_ctypes_structs_match_c_layout(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "preft.h"\n'
        "int main(void){\n"
        'printf("%zu %zu %zu %zu\\n", sizeof(preft_meta_t), offsetof(preft_meta_t, E_cap),'
        " offsetof(preft_meta_t, slot_split), sizeof(preft_lora_site_t));\n"
        'printf("%zu %zu %zu\\n", offsetof(preft_lora_site_t, bias), offsetof(preft_lora_site_t, ldy),'
        " offsetof(preft_lora_site_t, n));\n"
        'printf("%zu %zu %zu %zu\\n", sizeof(preft_xchg_t), offsetof(preft_xchg_t, part),'
        " offsetof(preft_xchg_t, state), offsetof(preft_xchg_t, spin_ns));\nreturn 0;}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    M, S = _lib.PreftMeta, _lib.PreftLoraSite
    assert [int(v) for v in out[:4]] == [ctypes.sizeof(M), M.E_cap.offset, M.slot_split.offset, ctypes.sizeof(S)]
    assert [int(v) for v in out[4:7]] == [S.bias.offset, S.ldy.offset, S.n.offset]
    X = _lib.PreftXchg
    assert [int(v) for v in out[7:]] == [ctypes.sizeof(X), X.part.offset, X.state.offset, X.spin_ns.offset]


def test_status_codes_map_to_reference_exceptions():
    assert isinstance(errors.status_to_error(1, "x"), errors.ShapeError)
    assert isinstance(errors.status_to_error(2, "x"), errors.RankError)
    assert isinstance(errors.status_to_error(5, "x"), errors.BatchError)
    assert isinstance(errors.status_to_error(7, "x"), errors.SyncError)
    assert isinstance(errors.status_to_error(8, "x"), errors.InfeasibleBatchError)
    assert isinstance(errors.status_to_error(16, "x"), errors.DeviceError)
    # same base classes as the reference (errors.py:1-5)
    assert issubclass(errors.StateError, RuntimeError) and issubclass(errors.BatchError, ValueError)


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("this check is for hosts without a GPU")
    import numpy as np

    from paper_2605_14217_b200 import AdapterKind, delta_for_rows, init_zero_delta
    from paper_2605_14217_b200.meta import BatchMeta

    with pytest.raises(errors.DeviceError):
        BatchMeta(4, 16)
    with pytest.raises(errors.DeviceError):
        delta_for_rows(init_zero_delta(AdapterKind.DIREFT, 2, (8,), seed=0), np.zeros((3, 8)))


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_2605_14217_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", text, flags=re.M), f
        assert "preft_oracle" not in text, f


def test_exchange_region_layout_host_side():
    """preft_xchg_init fills a rank's view of the fused kernel's exchange
    regions exactly as include/preft.h lays them out (host-only: no device
    memory is touched): partial planes, then the flags, then the state words."""
    lib = _lib.load()
    tp, planes, T_cap, U_cap = 4, 2, 96, 40
    nbytes = lib.preft_xchg_region_bytes(tp, planes, T_cap, U_cap)
    part = 2 * tp * planes * T_cap * 64 * 4
    flags = 2 * tp * planes * U_cap * 4
    assert nbytes >= part + flags + 64
    bases = [0x10000000 * (r + 1) for r in range(tp)]
    for rank in range(tp):
        xg = _lib.PreftXchg()
        arr = (ctypes.c_void_p * tp)(*bases)
        assert lib.preft_xchg_init(ctypes.byref(xg), arr, tp, rank, planes, T_cap, U_cap, 1) == 0
        assert (xg.tp_size, xg.tp_rank, xg.planes, xg.T_cap, xg.U_cap, xg.peer_sys) == (tp, rank, planes, T_cap, U_cap, 1)
        assert [xg.part[d] for d in range(tp)] == bases
        assert [xg.flag[d] for d in range(tp)] == [b + part for b in bases]
        assert xg.state == bases[rank] + part + flags
        assert xg.spin_ns > 0
    # invalid layouts are rejected without touching anything
    xg = _lib.PreftXchg()
    assert lib.preft_xchg_init(ctypes.byref(xg), (ctypes.c_void_p * 2)(bases[0], bases[1] + 4), 2, 0, 1, T_cap,
                               U_cap, 0) != 0  # misaligned peer base
    assert lib.preft_xchg_init(ctypes.byref(xg), (ctypes.c_void_p * 9)(*([bases[0]] * 9)), 9, 0, 1, T_cap, U_cap,
                               0) != 0  # more ranks than PREFT_XCHG_MAX_TP
