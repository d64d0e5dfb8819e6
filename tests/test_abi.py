"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/scqr3.h declares,
the ctypes structs match the header layout, and host-only entry points behave."""
import ctypes
import os
import re

import pytest

from paper_1809_11085_b200 import _abi, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "scqr3.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scqr3_[a-z_0-9]+)\s*\(", src)))


def test_library_builds_and_exports_every_header_symbol():
    build.build()
    lib = _abi.lib()
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_abi.EXPORTED) == names


def test_struct_layout_matches_header():
    # scqr3_pass_trace: double, int32, int32, double, double, double
    assert ctypes.sizeof(_abi.PassTrace) == 40
    # scqr3_opts field offsets (x86-64 SysV, as compiled from the header)
    o = _abi.Opts
    assert o.shift_value.offset == 8 and o.norm2_bound.offset == 24 and o.stop_tol.offset == 48
    assert o.m_global.offset == 56 and o.stream.offset == 64 and o.workspace.offset == 80
    assert o.prof.offset == 120 and o.trsm_diag.offset == 128   # ABI version 2 appends trsm_diag
    assert ctypes.sizeof(o) == 136
    assert ctypes.sizeof(_abi.Prof) == 96


def test_default_opts_and_sizes_without_gpu():
    lib = _abi.lib()
    o = _abi.Opts()
    lib.scqr3_default_opts(ctypes.byref(o))
    assert o.abi_version == _abi.SCQR3_ABI_VERSION and o.max_passes == 8 and o.stop_tol == 0.5
    assert o.power_iters == 32 and o.shift_mode == _abi.SHIFT_SAFE and o.norm_mode == _abi.NORM_POWER
    assert lib.scqr3_workspace_size(1000, 0, 0) == 0
    assert lib.scqr3_workspace_size(1000, 513, 0) == 0
    assert lib.scqr3_workspace_size(1000, 512, 0) > 0
    # complex X up to n = 512 (n > 256: the split matrix as two column blocks, zwide.cu)
    assert lib.scqr3_workspace_size_complex(1000, 0) == 0
    assert lib.scqr3_workspace_size_complex(1000, 513) == 0
    assert lib.scqr3_workspace_size_complex(1000, 512) > lib.scqr3_workspace_size_complex(1000, 256) > 0
    a = lib.scqr3_workspace_size(10_000_000, 128, 0)
    b = lib.scqr3_workspace_size(10_000_000, 128, 1)
    assert 0 < a < b and b >= 8 * 10_000_000 * 128       # oblique holds B*Q
    assert lib.scqr3_host_workspace_size(1000, 16) >= 8 * 1000 * 16


def test_invalid_arguments_fail_loudly_without_touching_a_gpu():
    lib = _abi.lib()
    o = _abi.Opts()
    lib.scqr3_default_opts(ctypes.byref(o))
    o.abi_version = 99
    assert lib.scqr3_factor(10, 2, None, 10, None, 10, None, ctypes.byref(o)) == _abi.EINVAL
    assert "abi_version" in _abi.last_error()
    lib.scqr3_default_opts(ctypes.byref(o))
    assert lib.scqr3_factor(10, 0, None, 10, None, 10, None, ctypes.byref(o)) == _abi.EINVAL
    assert lib.scqr3_factor(10, 300, None, 10, None, 10, None, ctypes.byref(o)) == _abi.EINVAL


def test_no_oracle_in_the_product_path():
    pkg = os.path.join(ROOT, "paper_1809_11085_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", text).lower() or f == "build.py", f


def test_header_enums_match_binding():
    import re
    hdr = open(os.path.join(ROOT, "include", "scqr3.h")).read()
    vals = {k: int(v) for k, v in re.findall(r"SCQR3_(\w+) = (\d+)", hdr)}
    for name in ["OK", "EINVAL", "EBREAKDOWN", "ENOCONV", "NORM_POWER", "NORM_FROBENIUS", "NORM_USER"]:
        assert vals[name] == getattr(_abi, name)
    for name in ["SAFE", "FIXED", "NONE", "ADAPTIVE", "PRACTICAL"]:
        assert vals["SHIFT_" + name] == getattr(_abi, "SHIFT_" + name)


def test_struct_layouts_against_the_compiled_header(tmp_path):
    """sizeof/offsetof of every ABI struct as gcc lays out include/scqr3.h, vs the ctypes mirror."""
    import subprocess
    fields = {"scqr3_opts": (_abi.Opts, "Opts"), "scqr3_pass_trace": (_abi.PassTrace, "PassTrace"),
              "scqr3_prof": (_abi.Prof, "Prof"), "scqr3_csr": (_abi.Csr, "Csr")}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "scqr3.h"', "int main(void) {"]
    for cname, (cls, _) in fields.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _t in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, (cls, _) in fields.items():
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for f, _t in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)
