"""Host-side checks of the C-ABI library (-m "not gpu"): it builds, loads, exports every
symbol include/nf.h declares, validates arguments, and refuses to run without a GPU
(there is no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nf():
    from paper_1902_06714_b200 import build
    build.build()
    import paper_1902_06714_b200 as nf
    return nf


def _declared():
    src = open(os.path.join(ROOT, "include", "nf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nf_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(nf):
    lib = ctypes.CDLL(nf.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(nf.EXPORTS)


def test_library_is_sm100a_device_code(nf):
    out = subprocess.run(["cuobjdump", "--list-elf", nf.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_validation(nf):
    with pytest.raises(nf.NFError) as e:
        nf.nf_net_create([784], "sigmoid")
    assert e.value.code == nf.NF_EINVAL
    with pytest.raises(nf.NFError) as e:
        nf.nf_net_create([3, 0, 2], "sigmoid")
    assert e.value.code == nf.NF_EINVAL
    with pytest.raises(nf.NFError) as e:
        nf.nf_net_create([3, 5, 2], "softmax")          # never a silent default
    assert e.value.code == nf.NF_EINVAL
    assert "softmax" in nf.nf_last_error()


def test_no_cpu_fallback_without_gpu(nf):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(nf.NFError) as e:
        nf.nf_net_create([3, 5, 2], "sigmoid")
    assert e.value.code == nf.NF_ENODEV


def test_binding_rejects_wrong_dtypes(nf):
    with pytest.raises(TypeError):
        nf._ptr(np.zeros(3, np.float64))
    with pytest.raises(TypeError):
        nf._ptr(np.zeros((3, 4), np.float32)[:, :2])


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1902_06714_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "__init__.py" and \
                    "import oracle" not in txt, f
