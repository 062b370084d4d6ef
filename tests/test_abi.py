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


def test_null_net_is_rejected_by_every_entry_point(nf):
    """Every call validates its handle before touching the device (no GPU needed)."""
    lib = nf.lib()
    null = None
    f = np.zeros(4, np.float32)
    p = f.ctypes.data_as(ctypes.c_void_p)
    assert lib.nf_set_stream(null, None) == nf.NF_EINVAL
    assert lib.nf_set_math(null, 0) == nf.NF_EINVAL
    assert lib.nf_param_count(null) == -1
    assert lib.nf_get_params(null, p, 4) == nf.NF_EINVAL
    assert lib.nf_set_params(null, p, 4) == nf.NF_EINVAL
    assert lib.nf_output(null, p, 1, p) == nf.NF_EINVAL
    assert lib.nf_train_batch(null, p, p, 1, 1.0) == nf.NF_EINVAL
    assert lib.nf_grad(null, p, p, 1, p) == nf.NF_EINVAL
    v = ctypes.c_float()
    assert lib.nf_loss(null, p, p, 1, ctypes.byref(v)) == nf.NF_EINVAL
    assert lib.nf_accuracy(null, p, p, 1, ctypes.byref(v)) == nf.NF_EINVAL
    st = np.zeros(1, np.int64)
    assert lib.nf_train_steps(null, p, p, 4, 1, st.ctypes.data_as(ctypes.c_void_p), 1, 1.0, None) == nf.NF_EINVAL
    lib.nf_net_destroy(null)                     # no-op
    assert lib.nf_launch_count() >= 0
    assert "null net" in nf.nf_last_error()


def test_create_rejects_bad_specs_before_the_device(nf):
    for dims, act in [([3, 5, 2], "relu,softmax"), ([3, 5, 2], "tanh,"), ([2, -1], "sigmoid"), ([], "sigmoid"),
                      ([3, 5, 4, 2], "relu,tanh,sigmoid,step"), ([3, 5, 4, 2], "relu,,sigmoid")]:
        with pytest.raises(nf.NFError) as e:
            nf.nf_net_create(dims, act)
        assert e.value.code == nf.NF_EINVAL, (dims, act)
    out = ctypes.c_void_p()
    d = np.array([3, 5, 2], np.int32)
    assert nf.lib().nf_net_create(d.ctypes.data_as(ctypes.c_void_p), 3, b"sigmoid", 0, None) == nf.NF_EINVAL


def test_header_documents_every_entry_point():
    """Each declaration in include/nf.h is preceded by a comment block (argument meaning,
    layout, ownership, errors) -- the boundary contract."""
    src = open(os.path.join(ROOT, "include", "nf.h")).read()
    for name in _declared():
        m = re.search(r"^[A-Za-z_][\w \*]*\b" + name + r"\(", src, flags=re.M)   # the declaration line
        assert m, name
        before = src[:m.start()].rstrip()
        assert before.endswith("*/"), name


def test_load_rejects_missing_and_malformed_files_before_the_device(nf, tmp_path):
    """nf_load validates the header, then the payload, before any device work; each kind of
    format error has its own code, never NF_ENODEV on this GPU-less host."""
    with pytest.raises(nf.NFError) as e:
        nf.nf_load(str(tmp_path / "missing.net"))
    assert e.value.code == nf.NF_EIO
    bad = [
        ("not a network\n", nf.NF_EFMT_MAGIC),
        ("nf-b200-net 7\n3\n3 5 2\nsigmoid\n", nf.NF_EFMT_VERSION),
        ("nf-b200-net 1\n3\n3 5 2\nsigmoid\n0.5\n", nf.NF_EFMT_TRUNCATED),    # 1 of 32 parameters
        ("nf-b200-net 1\n3\n3 0 2\nsigmoid\n", nf.NF_EFMT_DIMS),                # a zero width
        ("nf-b200-net 2\n3\n3 5 2\nsoftmax\nfp32\n", nf.NF_EFMT_ACTIVATION),
        ("nf-b200-net 2\n3\n3 5 2\nrelu,tanh,sigmoid\nfp32\n", nf.NF_EFMT_ACTIVATION),  # 3 names, 2 layers
        ("nf-b200-net 2\n3\n3 5 2\nsigmoid\nfp16\n", nf.NF_EFMT_PRECISION),
        ("nf-b200-net 2\n3\n3 5 2\nsigmoid\nfp64\n" + "0.5\n" * 31, nf.NF_EFMT_TRUNCATED),
    ]
    for i, (text, code) in enumerate(bad):
        path = tmp_path / f"bad{i}.net"
        path.write_text(text)
        with pytest.raises(nf.NFError) as e:
            nf.nf_load(str(path))
        assert e.value.code == code, text
    # a precision other than the requested one is rejected before the device, never narrowed
    path = tmp_path / "f64.net"
    path.write_text("nf-b200-net 2\n3\n3 5 2\nsigmoid\nfp64\n" + "0.1\n" * 32)
    with pytest.raises(nf.NFError) as e:
        nf.nf_load_as(str(path), nf.NF_MATH_FP32)
    assert e.value.code == nf.NF_EFMT_PRECISION
    path.write_text("nf-b200-net 2\n3\n3 5 2\nsigmoid\nfp32\n" + "0.5\n" * 32)
    with pytest.raises(nf.NFError) as e:
        nf.nf_load_as(str(path), nf.NF_MATH_FP64)
    assert e.value.code == nf.NF_EFMT_PRECISION
    # well-formed files get as far as the device (NF_ENODEV on a GPU-less host; loaded on a GPU box)
    import torch
    for math in (-1, nf.NF_MATH_FP32):
        if torch.cuda.is_available():
            nf.nf_net_destroy(nf.nf_load_as(str(path), math))
            continue
        with pytest.raises(nf.NFError) as e:
            nf.nf_load_as(str(path), math)
        assert e.value.code == nf.NF_ENODEV
