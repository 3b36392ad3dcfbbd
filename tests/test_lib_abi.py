"""The C-ABI library loads without a GPU and exports every symbol the public header declares.
No compute calls (CPU suite)."""

import ctypes
import os
import re

import pytest

from paper_2507_03220_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ss_b200.h")).read()
    return sorted(set(re.findall(r"SS_API\s+[\w\s\*]+?\b(ss_\w+)\s*\(", text)))


def test_header_declares_expected_symbols():
    syms = header_symbols()
    assert set(syms) == set(_lib.EXPORTED), syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.ss_version()


def test_struct_layout_matches_header():
    # 4 x u32 + (ptr, i64) x 3 = 16 + 48 bytes, natural alignment
    assert ctypes.sizeof(_lib.SsSeg) == 64
    assert _lib.SsSeg.src.offset == 16 and _lib.SsSeg.dst_base.offset == 48
    # ss_grad_seg: 4 x u32 + (ptr, i64) x 3 + 3 ptrs
    assert ctypes.sizeof(_lib.SsGradSeg) == 88
    assert _lib.SsGradSeg.x.offset == 16 and _lib.SsGradSeg.grad_a.offset == 64
    # ss_ipc_mem: 64-byte cudaIpcMemHandle_t + u64 offset + u64 bytes + i32 device + u32
    assert ctypes.sizeof(_lib.SsIpcMem) == 88 and _lib.SsIpcMem.offset.offset == 64
    assert ctypes.sizeof(_lib.SsIpcEvt) == 64


def test_ipc_calls_fail_cleanly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    ptr, mem = ctypes.c_void_p(), _lib.SsIpcMem()
    assert lib.ss_ipc_alloc(0, 1024, ctypes.byref(ptr), ctypes.byref(mem)) != _lib.SS_OK
    assert not ptr.value and lib.ss_ipc_last_error()
    assert lib.ss_ipc_export(None, 0, ctypes.byref(mem)) == _lib.SS_E_ARG


def test_context_creation_fails_cleanly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.ss_ctx_create(0, 0, 1, ctypes.byref(h))
    assert rc != _lib.SS_OK and not h.value


def test_null_context_is_rejected():
    lib = _lib.load()
    assert lib.ss_compute_batch(None, 0, 0, 0, 0, None, None, None) == _lib.SS_E_ARG
    assert lib.ss_kernel_launches(None) == -1
    assert lib.ss_last_error(None) == b"null context"


def test_executor_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2507_03220_b200 import GpuBaseExecutor
    with pytest.raises(RuntimeError):
        GpuBaseExecutor({})


def test_every_context_option_is_documented_in_the_header():
    """ss_set_option keys accepted by the library (ss_api.cu) all appear in the header's option
    list, so a binding author sees every knob and its default."""
    src = open(os.path.join(ROOT, "paper_2507_03220_b200", "csrc", "ss_api.cu")).read()
    keys = sorted(set(re.findall(r'strcmp\(key, "(\w+)"\)', src)))
    header = open(os.path.join(ROOT, "include", "ss_b200.h")).read()
    assert keys
    missing = [k for k in keys if not re.search(r"[\s,(]" + k + r"[\s,(]", header)]
    assert not missing, missing
