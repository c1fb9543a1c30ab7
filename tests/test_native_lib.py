"""CPU-side checks of the C ABI library: it was built for sm_100a, loads,
and exports every symbol include/remlot_b200.h declares (no compute calls
here -- there is no GPU in the build container)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1704_05132_b200 import _native

HEADER = os.path.join(ROOT, "include", "remlot_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(rl_\w+)\s*\(", text, re.M)))


def test_header_declares_python_exports():
    assert set(_declared()) == set(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_last_error_is_a_string():
    assert isinstance(_native.load().rl_last_error(), bytes)


def test_bad_arguments_rejected_without_gpu():
    lib = _native.load()
    h = ctypes.c_void_p()
    rc = lib.rl_instance_create(0, 5, *([None] * 8), ctypes.byref(h))
    assert rc == _native.RL_EINVAL
    assert b"bad arguments" in lib.rl_last_error()
    rc = lib.rl_list_moves(7, 4, *([None] * 9))
    assert rc == _native.RL_EINVAL
