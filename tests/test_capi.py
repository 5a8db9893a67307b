"""The C-ABI boundary on CPU: libasmc_b200.so loads, exports every symbol that
include/asmc_b200.h declares, the ctypes layouts in abi.py match the C structs
(sizes/offsets from a gcc-compiled probe), and the SASS carries sm_100a code.
No compute calls here (no GPU)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2408_12057_b200 import abi, capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "asmc_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(asmc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(capi.EXPORTED) <= set(names)


def test_struct_layouts_match_header(tmp_path):
    probe = tmp_path / "probe.c"
    probe.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "asmc_b200.h"\n'
                     "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu\\n\","
                     "sizeof(asmc_target_desc), sizeof(asmc_kernel_desc), sizeof(asmc_exec),"
                     "sizeof(asmc_logacc), sizeof(asmc_report), sizeof(asmc_rounds_out),"
                     "offsetof(asmc_report, log_z_hat), offsetof(asmc_exec, stream));return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(abi.TargetDesc), C.sizeof(abi.KernelDesc), C.sizeof(abi.Exec),
            C.sizeof(abi.LogAcc), C.sizeof(abi.Report), C.sizeof(abi.RoundsOut),
            abi.Report.log_z_hat.offset, abi.Exec.stream.offset]
    assert got == want


def test_no_device_means_no_samples():
    if capi.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(capi.AsmcError) as e:
        capi.run_sais_single(abi.gaussian_shift(0, 1, 1, 1), abi.kernel(), [0.0, 1.0], 16)
    assert e.value.code == abi.ERR_CUDA


def test_validation_codes_match_reference_exceptions():
    # argument checks run before any device access and map to the reference's classes
    with pytest.raises(capi.AsmcError) as e:
        capi.run_sais_single(abi.gaussian_shift(0, 1, 1, 1), abi.kernel(), [0.0, 0.5], 16)
    assert e.value.code == abi.ERR_INVALID_ARGUMENT and "end at beta = 1" in e.value.msg
    with pytest.raises(capi.AsmcError) as e:
        capi.run_sais_single(abi.mixture(2, .5, -1, .5, 1, .5, 2), abi.kernel(abi.KERNEL_IDEALIZED),
                             [0.0, 1.0], 16)
    assert e.value.code == abi.ERR_CAPABILITY
    assert capi.budget(16, 8, 1, 1 << 40, abi.MODE_SSMC) == (23, 12)


def test_kernels_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout
