"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/smc.h declares, reports its ABI version, and fails loudly (no
CPU fallback) when no CUDA device is present."""
import ctypes
import os
import re
import subprocess

import pytest

from tests.conftest import cuda_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "smc.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(smc_[a-z0-9_]+)\s*\(", src))
    # typedef'd function pointer fields are not exports
    return sorted(n for n in names if n not in {"smc_comm"})


def test_library_exports_every_declared_symbol():
    import paper_2112_00364_b200 as smc
    lib = ctypes.CDLL(smc._LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 24
    for name in syms:
        assert hasattr(lib, name), name
    # and nm agrees that they are dynamic text symbols with C linkage
    out = subprocess.run(["nm", "-D", "--defined-only", smc._LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (smc_[a-z0-9_]+)$", out, flags=re.M))
    assert set(syms) <= exported
    assert lib.smc_abi_version() == 2


def test_binding_covers_header():
    import paper_2112_00364_b200 as smc
    assert set(declared_symbols()) == set(smc.EXPORTED)


def test_library_is_sm100a():
    import paper_2112_00364_b200 as smc
    out = subprocess.run(["cuobjdump", "--list-elf", smc._LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(cuda_available(), reason="checks the no-device failure path")
def test_no_cpu_fallback():
    import inputs
    import paper_2112_00364_b200 as smc
    with pytest.raises(smc.SmcError) as e:
        smc.Smc(smc.Model.crbd(inputs.tree("tree5")), 100, 1)
    assert e.value.code in (smc.ECUDA, smc.EINVAL)


def test_invalid_arguments_rejected_before_device():
    import paper_2112_00364_b200 as smc
    # unknown kind and bad tree are rejected with EINVAL regardless of the device
    with pytest.raises(smc.SmcError) as e:
        smc.Smc(smc.Model(999), 10, 1)
    assert "unknown model kind" in str(e.value)
    with pytest.raises(smc.SmcError) as e:
        smc.Smc(smc.Model(smc.CRBD, [3.0, 0.0], None), 10, 1)
    assert "tree" in str(e.value)
    with pytest.raises(smc.SmcError) as e:
        smc.Resampler(100, state_bytes=24)
    assert "state_bytes" in str(e.value)
