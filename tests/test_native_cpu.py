"""The C-ABI library loads without a GPU, exports every symbol the public
header declares, and NVRTC accepts the generated elementwise sources for
every scalar kernel and dtype (compile only — no device work on CPU)."""
import os
import re

import pytest

from paper_1605_02688_b200 import codegen, native
from paper_1605_02688_b200.dtypes import FLOAT32, FLOAT64, INT32, INT64
from paper_1605_02688_b200.elemwise import KERNELS, EwProgram, kernel_out_dtype

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "texpr_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(tx_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_header_symbols():
    lib = native.library()
    assert lib.version() == 1
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib.lib, s), s
    assert set(syms) == set(native.EXPORTS)


def test_no_device_is_reported_not_faked():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    lib = native.library()
    from paper_1605_02688_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        lib.init(0)


@pytest.mark.parametrize("dt", [FLOAT32, FLOAT64, INT64])
def test_every_kernel_compiles_with_nvrtc(dt):
    lib = native.library()
    for k, spec in KERNELS.items():
        if dt == INT64 and k in ("sigmoid", "tanh", "exp", "log", "log1p", "sqrt"):
            ins = [dt] * spec.arity
        else:
            ins = [dt] * spec.arity
        if k == "switch":
            ins = ["bool", dt, dt]
        p = EwProgram.single(k, ins)
        assert lib.ew_check(codegen.generate_source(p)) > 0


def test_mixed_dtype_program_compiles():
    lib = native.library()
    # int32 * float32 + bool -> float32; comparison -> bool output
    nodes = [("mul", [("in", 0), ("in", 1)], kernel_out_dtype("mul", [INT32, FLOAT32])),
             ("add", [("node", 0), ("in", 2)], FLOAT32),
             ("gt", [("node", 1), ("const", 0)], "bool")]
    p = EwProgram([INT32, FLOAT32, "bool"], [(FLOAT32, 0.5)], nodes, [("node", 1), ("node", 2)])
    assert lib.ew_check(codegen.generate_source(p)) > 0


def test_literals_are_exact():
    import struct
    s = codegen.literal(FLOAT32, 0.13)
    bits = int(s.split("0x")[1].rstrip(")"), 16)
    assert struct.unpack("<f", struct.pack("<I", bits))[0] == struct.unpack("<f", struct.pack("<f", 0.13))[0]
