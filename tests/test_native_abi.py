"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
entry point declared in include/drivegrid_b200.h; the ctypes mirrors of the
ABI structs match the C layout byte for byte."""

from __future__ import annotations

import ctypes as ct
import re
import subprocess
from pathlib import Path

import pytest

from paper_2605_08528_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "drivegrid_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(dg_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert {"dg_create", "dg_destroy", "dg_step", "dg_observe", "dg_reset", "dg_check_actions",
            "dg_read_error", "dg_lane_follower", "dg_last_error", "dg_abi_version"} <= set(names)
    assert set(names) == set(N.SIGNATURES), "ctypes signature table out of sync with the header"


def test_library_loads_and_exports_every_symbol():
    lib = N.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.dg_abi_version() == N.ABI_VERSION
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported"


def test_library_targets_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("struct", ["DgDims", "DgConsts", "DgEngineDesc", "DgStepIO", "DgScenePool",
                                    "DgSceneBuild", "DgSceneSegments", "DgWorldBuild"])
def test_struct_layout_matches_c(struct, tmp_path):
    src = tmp_path / "sz.c"
    fields = [f for f, _ in getattr(N, struct)._fields_]
    body = "".join(f'printf("%zu ", offsetof({struct}, {f}));' for f in fields)
    src.write_text(f'#include <stdio.h>\n#include <stddef.h>\n#include "drivegrid_b200.h"\n'
                   f'int main(void){{ printf("%zu ", sizeof({struct})); {body} return 0; }}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    cls = getattr(N, struct)
    want = [ct.sizeof(cls)] + [getattr(cls, f).offset for f in fields]
    assert got == want


def test_create_rejects_bad_descriptions_without_a_gpu():
    lib = N.load_library()
    h = ct.c_void_p()
    assert lib.dg_create(None, ct.byref(h)) == N.DG_EINVAL
    d = N.DgEngineDesc()
    d.dims.W, d.dims.M = 1, 17
    assert lib.dg_create(ct.byref(d), ct.byref(h)) == N.DG_EINVAL
    assert b"M <= 16" in lib.dg_last_error()


def test_integration_stub_matches_the_binding():
    """The ctypes stub INTEGRATION.md hands a drivegrid maintainer declares
    the same struct fields (names, types, offsets) as this package's binding."""
    import re
    text = (N.ROOT / "INTEGRATION.md").read_text()
    block = next(b for b in re.findall(r"```python\n(.*?)```", text, re.S) if "class DgDims" in b)
    block = block.replace('ct.CDLL("libdrivegrid_b200.so")', f'ct.CDLL({str(N.LIB_PATH)!r})')
    ns = {"CONST_FIELDS": N.CONST_FIELDS}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    for name in ("DgDims", "DgConsts", "DgEngineDesc", "DgStepIO"):
        stub, ours = ns[name], getattr(N, name)
        assert [f[0] for f in stub._fields_] == [f[0] for f in ours._fields_], name
        assert ct.sizeof(stub) == ct.sizeof(ours), name
        for f, _ in ours._fields_:
            assert getattr(stub, f).offset == getattr(ours, f).offset, (name, f)


def test_world_build_rejects_bad_arguments_without_a_gpu():
    lib = N.load_library()
    assert lib.dg_build_scenes(None, None, None, None) == N.DG_EINVAL
    pool, seg, b = N.DgScenePool(), N.DgSceneSegments(), N.DgWorldBuild()
    assert lib.dg_build_worlds(ct.byref(pool), ct.byref(seg), ct.byref(b), None) == N.DG_EINVAL
    assert b"bad dimensions" in lib.dg_last_error()
