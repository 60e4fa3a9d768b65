"""The reciprocal-based division used by the spectral criterion kernel
(csrc/kernels/exact_div.cuh) must be bitwise IEEE division: 2^27 random
operand pairs per exponent regime, compared with __ddiv_rn on the device."""
import ctypes
import os
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
KDIR = os.path.join(os.path.dirname(HERE), "paper_2306_10025_b200", "csrc", "kernels")


@pytest.mark.gpu
@pytest.mark.parametrize("regime", [0, 1, 2, 3])
def test_div_rn_recip_is_ieee_division(regime):
    with tempfile.TemporaryDirectory() as td:
        so = os.path.join(td, "exact_div_check.so")
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false", "-shared",
                               "-Xcompiler", "-fPIC", "-I", KDIR, "-o", so,
                               os.path.join(HERE, "cuda", "exact_div_check.cu")])
        lib = ctypes.CDLL(so)
        lib.exact_div_check.restype = ctypes.c_ulonglong
        lib.exact_div_check.argtypes = [ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int]
        for seed in (1, 2):
            assert lib.exact_div_check(1 << 27, seed * 7919 + regime, regime) == 0
