"""The C ABI: libdockscreen.so loads and exports every symbol include/dockscreen.h declares,
and the ctypes struct mirrors have the header's sizes.  No compute calls (CPU-only)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2209_05069_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "dockscreen.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w ]+?\**\s*\b(ds_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_loads_and_exports_every_declared_symbol():
    L = native.lib()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (ds_\w+)", out))
    assert set(names) <= exported


def test_struct_layouts_match_header():
    """Compile a probe against the header and compare sizeof/offsetof with the ctypes mirrors."""
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "dockscreen.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(ds_pocket_desc), sizeof(ds_dock_config), sizeof(ds_batch_desc),
        sizeof(ds_result), sizeof(ds_restart_record), sizeof(ds_outputs), sizeof(ds_stats));
 printf("%zu %zu %zu %zu %zu\n", offsetof(ds_pocket_desc, n_bins), offsetof(ds_dock_config, seed),
        offsetof(ds_result, poses_scored), offsetof(ds_stats, h2d_bytes), offsetof(ds_stats, lat_spread));
 return 0;}
'''
    tmp = os.path.join(ROOT, "build")
    os.makedirs(tmp, exist_ok=True)
    src, exe = os.path.join(tmp, "abi_probe.c"), os.path.join(tmp, "abi_probe")
    open(src, "w").write(probe)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
    l1, l2 = subprocess.check_output([exe], text=True).split("\n")[:2]
    sizes = [int(x) for x in l1.split()]
    assert sizes == [C.sizeof(native.PocketDesc), C.sizeof(native.DockConfigC), C.sizeof(native.BatchDesc),
                     native.RESULT_DTYPE.itemsize, native.RESTART_DTYPE.itemsize, C.sizeof(native.Outputs),
                     C.sizeof(native.Stats)]
    offs = [int(x) for x in l2.split()]
    assert offs == [native.PocketDesc.n_bins.offset, native.DockConfigC.seed.offset,
                    native.RESULT_DTYPE.fields["poses_scored"][1], native.Stats.h2d_bytes.offset,
                    native.Stats.lat_spread.offset]


def test_kernels_are_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump), i.e. the device path is native code."""
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_is_a_loud_error():
    """Without a GPU every docking entry point fails loudly (no CPU fallback)."""
    if native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(native.NativeUnavailable):
        native.Context(0)
