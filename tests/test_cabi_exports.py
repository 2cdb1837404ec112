"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/spmvcomp_b200.h declares, and fails loudly (no CPU fallback) when
there is no CUDA device."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "spmvcomp_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spmvb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1612_00530_b200 import _cabi
    decl = declared_symbols()
    assert len(decl) >= 30
    missing = [s for s in decl if not hasattr(_cabi.lib, s)]
    assert not missing, missing
    assert sorted(_cabi.SYMBOLS) == decl


def test_status_codes_match_reference_taxonomy():
    from paper_1612_00530_b200 import _cabi
    text = open(os.path.join(ROOT, "include", "spmvcomp_b200.h")).read()
    for name, cls in (("INVALID_ARGUMENT", _cabi.InvalidArgument), ("TABLE_OVERFLOW", _cabi.TableOverflowError),
                      ("INTEGRITY", _cabi.IntegrityError), ("VERIFICATION", _cabi.VerificationError),
                      ("IO", _cabi.IoError), ("DIVERGENCE", _cabi.DivergenceError), ("CUDA", _cabi.CudaError)):
        code = int(re.search(rf"SPMVB_ERR_{name}\s*=\s*(\d+)", text).group(1))
        assert cls.code == code


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import paper_1612_00530_b200 as sp
    with pytest.raises(sp.CudaError):
        sp.device_count()
    with pytest.raises(sp.SpmvcompError):
        sp.upload_ell(1, 1, 1, np.array([26.0]), np.array([0], dtype=np.int32))
    with pytest.raises(sp.SpmvcompError):
        sp.generate_matrix(sp.GridSpec(2, 2, 2))
    with pytest.raises(sp.InvalidArgument):  # argument checks still come first (grid.hpp:35-47)
        sp.generate_matrix(sp.GridSpec(0, 1, 1))


def test_default_library_rejects_unknown_and_lab_options():
    """Measurement-only kernel variants (some return wrong y on purpose) are compiled only into the lab build;
    the default library must refuse the option values that select them, and unknown keys."""
    import paper_1612_00530_b200 as sp
    assert sp.get_option("lab_build") == 0
    with pytest.raises(sp.InvalidArgument):
        sp.set_option("no_such_option", 1)
    for key, values in (("box_march", (1, 5, 20, 47, 62, 96, 97, 98, 99, 100, 104, 118, 119, 120)), ("debug_nochain", (1, 7)),
                        ("ell_kernel", (4, 5, 6, 7)), ("pattern_kernel", (4, -1))):
        for v in values:
            with pytest.raises(sp.InvalidArgument):
                sp.set_option(key, v)
        assert sp.get_option(key) == 0
    for key, values in (("box_march", (3, 90, 101, 107, 108, 109, 110, 0)), ("ell_kernel", (1, 2, 3, 0)), ("pattern_kernel", (1, 2, 3, 0))):
        for v in values:
            sp.set_option(key, v)
            assert sp.get_option(key) == v


def test_default_library_holds_no_lab_kernels():
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    from paper_1612_00530_b200 import _cabi
    out = subprocess.run(["cuobjdump", "-elf", _cabi.SO_PATH], capture_output=True, text=True).stdout
    kernels = set(re.findall(r"^\.text\.(\S+)", out, flags=re.M))
    assert 0 < len(kernels) < 80, len(kernels)
    assert not [k for k in kernels if "box5" in k or "box6" in k or "box7" in k or "box8" in k]


def test_product_never_imports_the_oracle():
    """The oracle is test infrastructure: nothing under the product package may import,
    load, link or include it."""
    pkg = os.path.join(ROOT, "paper_1612_00530_b200")
    bad = re.compile(r"(^\s*(from|import)\s+oracle\b|liboracle|spmvcomp_oracle|oracle/|oracle\.py)", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")) or f == "Makefile":
                text = open(os.path.join(dirpath, f)).read()
                assert not bad.search(text), os.path.join(dirpath, f)
