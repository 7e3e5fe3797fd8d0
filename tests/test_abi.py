"""The C-ABI library loads and exports every entry point include/cdr.h
declares; without a device it fails loudly (no CPU fallback)."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2103_15208_b200 import api, build


def test_library_builds_and_exports_every_symbol():
    lib = build.build()
    assert os.path.exists(lib)
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    declared = set(api.exported_symbols())
    assert declared, "no cdr_* declarations found in include/cdr.h"
    assert declared <= exported, f"missing: {sorted(declared - exported)}"
    assert {s for s in exported if not s.startswith("cdr_")} == set()
    L = api.load_library()
    assert L.cdr_abi_version() == 2


def test_sm100a_cubin_embedded():
    lib = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    L = api.load_library()
    n = C.c_int(-1)
    L.cdr_device_count(C.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    assert L.cdr_create(0, C.byref(h)) == 6  # CDR_ERR_NO_DEVICE
    with pytest.raises(api.CollodiffError):
        api.Renderer(0)


def test_null_context_is_rejected():
    L = api.load_library()
    assert L.cdr_update_positions(None, None) == 5  # CDR_ERR_INVALID_ARG
    assert L.cdr_loss_grad(None, None, 0, None, 0.0, 0.0, 0, 0, None, None, None, None, None, None) == 5
