"""The C-ABI library loads and exports every entry point include/harl_b200.h
declares (no device needed: nothing is called)."""

import ctypes
import os
import re

import pytest

from paper_2211_11172_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "harl_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(harl_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_the_binding_binds():
    assert header_functions() == sorted(N.EXPORTED)


def header_prototypes():
    """{name: [param type strings]} from the header's declarations."""
    text = open(os.path.join(ROOT, "include", "harl_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(harl_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;", text):
        args = " ".join(m.group(2).split())
        out[m.group(1)] = [] if args in ("", "void") else args.split(",")
    return out


def _kind(decl):
    d = decl.strip()
    if "*" in d:
        return "ptr"
    if "int64_t" in d or "long long" in d:
        return "i64"
    if "double" in d:
        return "f64"
    return "i32"


def _ctkind(t):
    if t in (ctypes.c_void_p, ctypes.c_char_p) or hasattr(t, "_type_") and \
            not isinstance(t._type_, str):
        return "ptr"
    return {ctypes.c_int64: "i64", ctypes.c_longlong: "i64",
            ctypes.c_uint64: "i64", ctypes.c_ulonglong: "i64",
            ctypes.c_double: "f64"}.get(t, "i32")


def test_binding_signatures_match_the_header():
    protos = header_prototypes()
    for name, (_, args) in N._SIGS.items():
        want = [_kind(a) for a in protos[name]]
        got = [_ctkind(a) for a in args]
        assert got == want, name


def test_library_exports_every_symbol():
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("native library not built (run build())")
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in header_functions():
        assert hasattr(lib, name), name
    lib.harl_abi_version.restype = ctypes.c_int
    assert lib.harl_abi_version() == 1


STRUCTS = {"harl_sketch_desc": N.SketchDesc, "harl_pcg64": N.Pcg64,
           "harl_mlp_desc": N.MlpDesc, "harl_forest_desc": N.ForestDesc,
           "harl_replay_ring": N.ReplayRing, "harl_entry_log": N.EntryLog,
           "harl_track_stats": N.TrackStats,
           "harl_step_buffers": N.StepBuffers,
           "harl_net_layout": N.NetLayout, "harl_ppo_hyper": N.PpoHyper,
           "harl_copy_op": N.CopyOp}


def test_ctypes_layouts_match_the_c_compiler(tmp_path):
    """Compile a probe against the header and compare every field offset
    and struct size with the ctypes mirror."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lines = ['#include <stdio.h>', '#include <stddef.h>',
             '#include "harl_b200.h"', "int main(void){"]
    for cname, py in STRUCTS.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", '
                         f'offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True,
                         text=True).stdout.split("\n")
    got = dict(line.split() for line in out if line.strip())
    for cname, py in STRUCTS.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, \
                f"{cname}.{fname}"


def test_device_entry_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2211_11172_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        N.load(require_device=True)
