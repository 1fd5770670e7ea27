"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a,
loads, and exports every entry point include/vrp_rpd.h declares; the product
path refuses to run without a GPU (no CPU fallback)."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2602_23685_b200 import _native
from paper_2602_23685_b200 import build as B

REPO = Path(__file__).resolve().parent.parent
HEADER = REPO / "include" / "vrp_rpd.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(vrp_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def libpath():
    return B.build()


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "vrp_makespan_batch" in syms and "vrp_decode_batch" in syms
    assert len(syms) >= 8


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", str(libpath)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vrp_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", str(libpath)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_library_loads_and_reports_version(libpath):
    L = _native.lib(require_device=False)
    abi, arch = ctypes.c_int32(), ctypes.c_int32()
    assert L.vrp_version(ctypes.byref(abi), ctypes.byref(arch)) == 0
    assert abi.value >= 1 and arch.value == 1000


def test_null_arguments_are_rejected_without_device(libpath):
    L = _native.lib(require_device=False)
    rc = L.vrp_makespan_batch(None, None, 4, 0, None, 1, 0, None, None, None, None, None)
    assert rc == 1
    assert b"null" in L.vrp_last_error()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_gpu():
    from paper_2602_23685_b200.instance import FleetConfig, Instance
    from paper_2602_23685_b200.schedule import Solution, exact_makespan
    inst = Instance(n=1, d=((0, 10), (10, 0)), p=(0, 20), fleet=FleetConfig(1, 1), label="t")
    with pytest.raises(_native.NativeUnavailable):
        exact_makespan(inst, Solution.from_lists([[(1, "D"), (1, "P")]]))


def test_struct_layouts_match_python_mirrors(tmp_path):
    """sizeof / offsetof of the header's structs (compiled with gcc) equal the
    numpy dtypes and ctypes structures the Python side packs them with."""
    from paper_2602_23685_b200 import device as DV
    from paper_2602_23685_b200 import rng as R
    src = tmp_path / "sz.c"
    fields = ["z", "z_best", "temperature", "t_init", "weights", "scores", "attempts", "stagnation",
              "accepted", "rejected", "reheats", "best_it", "n_trace", "n_rows"]
    pfields = [f for f, _ in DV.AlnsParamsC._fields_]
    body = ['#include <stdio.h>', '#include <stddef.h>', '#include "vrp_rpd.h"', 'int main(void) {',
            'printf("%zu %zu %zu\\n", sizeof(vrp_philox), sizeof(vrp_alns_worker), sizeof(vrp_alns_params));']
    body += [f'printf("%zu\\n", offsetof(vrp_alns_worker, {f}));' for f in fields]
    body += [f'printf("%zu\\n", offsetof(vrp_alns_params, {f}));' for f in pfields]
    body += ['printf("%zu %zu %zu\\n", offsetof(vrp_philox, buffer_pos), offsetof(vrp_philox, has_uint32), '
             'offsetof(vrp_philox, uinteger));', 'return 0; }']
    src.write_text("\n".join(body))
    exe = tmp_path / "sz"
    subprocess.run(["gcc", f"-I{REPO / 'include'}", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    vals = [int(x) for x in out]
    assert vals[:3] == [R._DTYPE.itemsize, DV.ALNS_WORKER_DTYPE.itemsize, ctypes.sizeof(DV.AlnsParamsC)]
    k = 3
    for f in fields:
        assert vals[k] == DV.ALNS_WORKER_DTYPE.fields[f][1], f
        k += 1
    for f in pfields:
        assert vals[k] == getattr(DV.AlnsParamsC, f).offset, f
        k += 1
    assert vals[k:] == [R._DTYPE.fields[f][1] for f in ("buffer_pos", "has_uint32", "uinteger")]


def test_instance_size_limits_checked_before_any_device_work(libpath):
    """vrp_instance_create rejects n beyond VRP_MAX_N (the tightest per-kernel
    shared-memory bound) and m beyond 32 with VRP_EUNSUPPORTED, before it
    reads the matrices or touches a device -- so this runs on the CPU."""
    text = HEADER.read_text()
    max_n = int(re.search(r"#define VRP_MAX_N (\d+)", text).group(1))
    unsupported = int(re.search(r"#define VRP_EUNSUPPORTED (\d+)", text).group(1))
    lib = ctypes.CDLL(str(libpath))
    lib.vrp_instance_create.argtypes = [ctypes.c_int32] * 3 + [ctypes.c_void_p] * 3
    lib.vrp_last_error.restype = ctypes.c_char_p
    one = np.zeros(1)
    h = ctypes.c_void_p()
    for n, m in ((max_n + 1, 6), (0, 6), (10, 33)):
        rc = lib.vrp_instance_create(n, m, 1, one.ctypes.data, one.ctypes.data, ctypes.byref(h))
        assert rc == unsupported, (n, m, rc)
        assert b"must lie in" in lib.vrp_last_error()
