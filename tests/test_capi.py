"""The C-ABI library loads and exports every symbol include/*.h declares; with
no GPU it fails loudly with a status code (no CPU fallback, no crash)."""
import ctypes as C
import os
import re

import pytest

from paper_1902_07554_b200 import gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sbdt_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sbdt_gpu_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("sbdt_gpu_create", "sbdt_gpu_assign_points", "sbdt_gpu_assign_points_dev", "sbdt_gpu_find_border",
              "sbdt_gpu_find_border_dev", "sbdt_gpu_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(gpu.lib_path())
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_sm100a_code_present():
    # the fatbin must carry sm_100a SASS (built with -gencode arch=compute_100a,code=sm_100a)
    data = open(gpu.lib_path(), "rb").read()
    assert b"sm_100a" in data


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gpu.SbdtGpuError):
        gpu.Context(0)


def test_product_path_never_loads_the_oracle():
    import sys
    import subprocess
    code = ("import sys; import paper_1902_07554_b200 as p; p.gpu.lib(); "
            "assert not any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules), 'oracle imported'")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT)
    for f in ("gpu.py", "host.py", "__init__.py", "dist.py"):
        txt = open(os.path.join(ROOT, "paper_1902_07554_b200", f)).read()
        assert "import oracle" not in txt and "liboracle" not in txt
