"""CPU-side checks of the C-ABI boundary: libkc.so builds for sm_100a, loads
without a GPU, and exports every entry point include/kc.h declares; the
binding's struct layouts match the header; host-only logic (tracker errors
without a device) behaves."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kc.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kc_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def kclib():
    from paper_2605_03208_b200 import build, kc
    build.build_lib()
    return kc


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ["kc_track", "kc_capture", "kc_restore", "kc_replay", "kc_validate", "kc_hash", "kc_diff"]:
        assert must in names


def test_library_exports_every_declared_symbol(kclib):
    L = kclib.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert sorted(kclib.exported_symbols()) == _declared()
    out = subprocess.check_output(["nm", "-D", "--defined-only", kclib.LIB_PATH], text=True)
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_has_no_libcuda_link_dependency(kclib):
    out = subprocess.check_output(["ldd", kclib.LIB_PATH], text=True)
    assert "libcuda.so" not in out


def test_sm100a_code_in_library(kclib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", kclib.LIB_PATH], text=True)
    assert "sm_100a" in out


def _sass_of(lib_path, needle):
    out = subprocess.check_output(["cuobjdump", "-sass", lib_path], text=True)
    funcs, cur = {}, None
    for line in out.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return {k: "\n".join(v) for k, v in funcs.items() if needle in k}


def test_k1_staging_instructions_in_sass(kclib):
    # default K1 stages slices with cp.async (SASS LDGSTS); the TMA ring variant
    # uses cp.async.bulk (UBLKCP) + mbarriers (SYNCS); both use the fast round
    cp = _sass_of(kclib.LIB_PATH, "k1_hash_cpasync")
    tma = _sass_of(kclib.LIB_PATH, "k1_hash_tma")
    assert cp and all("LDGSTS" in s for s in cp.values())
    assert tma and all("UBLKCP" in s and "SYNCS" in s for s in tma.values())
    assert all("SHF.L.W" in s for s in cp.values())  # funnel-shift rotate of the XXH64 round


def test_k2_uses_256bit_loads(kclib):
    k2 = _sass_of(kclib.LIB_PATH, "k2_diff")
    assert k2 and all(".256" in s for s in k2.values())


def test_abi_version_and_status_strings(kclib):
    assert kclib.abi_version() == 1
    assert kclib.status_name(-6) == "KC_ERR_VA_UNAVAILABLE"
    assert "sm_100a" in kclib.build_info()


def test_struct_sizes_match_header(kclib):
    # sizes fixed by include/kc.h (x86-64 SysV layout)
    assert ctypes.sizeof(kclib.Region) == 32
    assert ctypes.sizeof(kclib.Buffer) == 40
    assert ctypes.sizeof(kclib.Tolerance) == 24
    assert ctypes.sizeof(kclib.DiffReport) == 14 * 8 + 8
    assert ctypes.sizeof(kclib.Dispatch) == 96
    assert ctypes.sizeof(kclib.Options) == 24
    assert ctypes.sizeof(kclib.CaptureReport) == 9 * 8 + 5 * 8
    assert ctypes.sizeof(kclib.ReplayOpts) == 80
    assert ctypes.sizeof(kclib.RestoreReport) == 6 * 8 + 4 * 8


def test_count_chunks_host_helper(kclib):
    regs = [(0x1000, 1), (0x20000, 65536), (0x100000, 65537), (0x300000, 3 * 65536 - 1)]
    assert kclib.count_chunks(regs) == 1 + 1 + 2 + 3
