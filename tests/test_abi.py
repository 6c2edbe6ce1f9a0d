"""CPU: the C-ABI library loads and exports exactly what include/hod.h declares.

No compute calls (no GPU here); the GPU tests exercise every entry point.
"""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hod.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hod_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2312_03549_b200.build_native import LIB, build

    build()  # no-op when up to date
    return ctypes.CDLL(str(LIB))


def test_header_declares_the_survey_boundary():
    names = declared()
    for required in ("hod_pack_bf16", "hod_sumsq_bf16", "hod_adamw_bf16", "hod_nccl_unique_id",
                     "hod_nccl_comm_init", "hod_reduce_scatter_bf16", "hod_all_gather_bf16",
                     "hod_all_reduce_f32", "hod_comm_destroy", "hod_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2312_03549_b200 import _native

    assert sorted(_native.EXPORTED) == declared()


def test_abi_version_and_error_slot(lib):
    lib.hod_abi_version.restype = ctypes.c_int
    assert lib.hod_abi_version() == 3
    lib.hod_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.hod_last_error(), bytes)


def test_argument_validation_without_gpu(lib):
    """Host-side validation fails before any CUDA call."""
    from paper_2312_03549_b200 import _native as nat

    L = nat.load()
    assert L.hod_pack_bf16(None, 0, None, 16, ctypes.c_float(1.0), 0, None) == 10001
    assert b"bad arguments" in L.hod_last_error()
    hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 0)
    assert L.hod_adamw_bf16(1, 1, 1, 1, 1, 16, ctypes.byref(hp), None, None) == 10001
    assert b"step" in L.hod_last_error()


def test_built_for_sm100a_only():
    import subprocess

    from paper_2312_03549_b200.build_native import LIB

    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, out.stdout


def test_struct_layouts_match_c(tmp_path):
    """ctypes mirrors of the ABI structs have the C sizes and field offsets."""
    import shutil
    import subprocess

    from paper_2312_03549_b200 import _native as nat

    gxx = shutil.which("g++") or "/usr/bin/g++"
    fields = {"hod_p2p_span": (nat.P2PSpan, ["local_grad", "master", "partials", "err", "bucket_start",
                                             "shard_numel", "n_buckets", "keep_reduced", "slot",
                                             "epoch", "tag", "timeout_ns"]),
              "hod_pack_entry": (nat.PackEntry, ["src", "numel", "dst_offset"]),
              "hod_adamw_params": (nat.AdamWParams, ["lr", "weight_decay", "step", "mode"])}
    lines = ['#include <cstdio>', '#include <cstddef>', '#include "hod.h"', "int main() {"]
    for cname, (_, names) in fields.items():
        lines.append(f'  printf("%zu\\n", sizeof({cname}));')
        for f in names:
            lines.append(f'  printf("%zu\\n", offsetof({cname}, {f}));')
    lines.append("}")
    src = tmp_path / "layout.cpp"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    r = subprocess.run([gxx, f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip(f"no C++ compiler: {r.stderr[:200]}")
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = []
    for _, (cls, names) in fields.items():
        want.append(ctypes.sizeof(cls))
        want += [getattr(cls, f).offset for f in names]
    assert got == want
