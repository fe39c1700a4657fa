"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/*.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1305_6738_b200 import _build, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "zipfks_b200.h")).read()
    return sorted(set(re.findall(r"\b(zks_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.load()


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert getattr(lib, name) is not None, name


def test_abi_version(lib):
    assert lib.zks_version() == _native.ABI_VERSION


def test_cell_struct_layout():
    assert ctypes.sizeof(_native.ZksCell) == 56
    assert _native.ZksCell.gamma.offset == 8
    assert _native.ZksCell.count.offset == 48


def test_cubin_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_invalid_arguments_fail_loudly_without_a_device(lib):
    # argument validation happens before any CUDA call
    rc = lib.zks_engine_create(0, None, 0, ctypes.byref(ctypes.c_void_p()))
    assert rc == _native.ZKS_EINVAL
    assert b"log table" in lib.zks_last_error()


def test_plain_c_consumer_links_and_runs(lib, tmp_path):
    # the header is plain C and the library links into a C program (the FFI a non-Python
    # host would use); only calls that need no device
    src = tmp_path / "consumer.c"
    src.write_text(
        '#include <stdio.h>\n#include "zipfks_b200.h"\n'
        "int main(void) {\n"
        "  zks_engine* e = 0;\n"
        "  double logs[2] = {0.0, 0.0};\n"
        "  int rc = zks_engine_create(0, logs, 2, &e);  /* rejected: logs_len < 65537 */\n"
        '  printf("%d %d %s\\n", zks_version(), rc != 0, zks_last_error());\n'
        "  return 0;\n}\n")
    exe = tmp_path / "consumer"
    libdir = os.path.dirname(_build.LIB)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L", libdir, "-l:" + os.path.basename(_build.LIB), "-Wl,-rpath," + libdir], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split(maxsplit=2)
    assert int(out[0]) == _native.ABI_VERSION and out[1] == "1" and "65537" in out[2]
