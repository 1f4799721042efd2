"""libfsp.so loads and exports every symbol include/fsp.h declares (no GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libfsp():
    from paper_1208_3933_b200 import build, binding
    build.build()
    return binding.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fsp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsp_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_1208_3933_b200 import binding
    assert declared_symbols() == sorted(binding.EXPORTS)


def test_every_symbol_exported(libfsp):
    for name in declared_symbols():
        assert hasattr(libfsp, name), name


def test_version_and_errors(libfsp):
    assert libfsp.fsp_version() == 1
    out = ctypes.c_void_p()
    # null ptm -> EINVAL without touching the device
    assert libfsp.fsp_instance_load(None, 5, 3, ctypes.byref(out)) == -1
    assert b"null" in libfsp.fsp_last_error()
    assert libfsp.fsp_lb_eval(None, None, 1, None, 0, None, None) == -1


def test_lb_work_formula(libfsp):
    # W(d) = 2dm + n'(3m-2) + n'm + P n + 4 P n' + 2P
    for n, m, d in [(200, 20, 100), (20, 5, 0), (500, 20, 499), (20, 20, 20)]:
        P, np_ = m * (m - 1) // 2, n - d
        w = 2 * d * m + np_ * (3 * m - 2) + np_ * m + P * n + 4 * P * np_ + 2 * P
        assert libfsp.fsp_lb_work(n, m, d) == w
    assert libfsp.fsp_lb_work(200, 20, 100) == 126180


def test_product_does_not_import_oracle():
    import subprocess, sys
    code = ("import sys; import paper_1208_3933_b200.binding, paper_1208_3933_b200.inputs;"
            "print(any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules))")
    out = subprocess.check_output([sys.executable, "-c", code], cwd=ROOT, text=True)
    assert out.strip() == "False"
    for root, _, files in os.walk(os.path.join(ROOT, "paper_1208_3933_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt, f
