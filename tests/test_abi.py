"""The C-ABI boundary (no GPU needed): libkpm.so loads, exports exactly the
entry points include/kpm.h declares, and the ctypes table binds all of them."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "kpm.h")
LIB = os.path.join(REPO, "paper_1905_09758_b200", "libkpm.so")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kpm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("kpm_init", "kpm_graph_from_edges", "kpm_graph_from_csr", "kpm_csr_matvec",
                 "kpm_run_create", "kpm_run_advance", "kpm_run_result", "kpm_dos_contrib",
                 "kpm_ldos", "kpm_filter_probes", "kpm_probes_rademacher", "kpm_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail("libkpm.so is not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (kpm_[a-z0-9_]+)$", out, flags=re.M))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for n in _declared():
        assert getattr(lib, n) is not None


def test_ctypes_table_covers_header():
    from paper_1905_09758_b200 import _lib
    assert sorted(_lib.SIGNATURES) == _declared()
    lib = _lib.load()
    assert lib.kpm_abi_version() == 1


def test_no_device_is_reported_not_faked():
    from paper_1905_09758_b200 import _lib
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.KpmLibraryError):
        _lib.Context(0)


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout


def test_host_prefault_is_host_only_and_bounds_safe():
    """kpm_host_prefault pages in caller buffers (aligned or not, tiny or
    multi-page, any thread count) without a GPU and rejects negative sizes."""
    import numpy as np

    from paper_1905_09758_b200 import _lib

    for nbytes, off in ((1, 0), (4095, 1), (4097, 3), (1 << 22, 5), ((1 << 22) + 7, 0)):
        buf = np.full(nbytes + off, 7, dtype=np.uint8)[off:]
        for th in (0, 1, 3, 16):
            _lib.prefault(buf, th)
        assert buf[0] == 0 and np.all(buf[buf != 0] == 7)
    empty = np.empty(0)
    _lib.prefault(empty)
    assert _lib.load().kpm_host_prefault(None, 0, 0) == 0
    assert _lib.load().kpm_host_prefault(empty.ctypes.data, -1, 0) != 0
