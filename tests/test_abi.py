"""The C-ABI library (no GPU needed): it loads, exports every function include/dog.h declares, validates
arguments before touching the device, and the Python binding keeps the C names.  No compute calls."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dog.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(dog_[a-z_]+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1605_02406_b200 import build
    build.build()
    return C.CDLL(build.LIB)


def test_header_parses():
    names = declared_functions()
    for must in ("dog_create", "dog_step", "dog_read_cells", "dog_destroy", "dog_get_state", "dog_set_state",
                 "dog_get_debug", "dog_step_host", "dog_error_string"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1605_02406_b200", "libdog.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (dog_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    for n in declared_functions():
        getattr(lib, n)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_1605_02406_b200", "libdog.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_uses_c_names():
    from paper_1605_02406_b200 import dog
    for n in declared_functions():
        assert hasattr(dog, n), n


def test_argument_validation_without_device(lib):
    from paper_1605_02406_b200 import dog
    g = dog.dog_grid(0, 10, 0.1)
    p = dog.dog_params(0.99, 0.02, 0.02, 0.8, 4.0, 2.0, 1.0, 0.0)
    h = C.c_void_p()
    assert dog.dog_create(C.byref(g), 100, 10, C.byref(p), 1, 0, 0, None, C.byref(h)) == dog.DOG_E_INVAL
    g = dog.dog_grid(16, 16, 0.1)
    bad = dog.dog_params(1.5, 0.02, 0.02, 0.8, 4.0, 2.0, 1.0, 0.0)
    assert dog.dog_create(C.byref(g), 100, 10, C.byref(bad), 1, 0, 0, None, C.byref(h)) == dog.DOG_E_INVAL
    bad = dog.dog_params(0.99, 0.02, 0.02, 0.8, 4.0, -2.0, 1.0, 0.0)
    assert dog.dog_create(C.byref(g), 100, 10, C.byref(bad), 1, 0, 0, None, C.byref(h)) == dog.DOG_E_INVAL
    g = dog.dog_grid(65535, 32769, 0.1)   # C >= 2^31 - 1
    assert dog.dog_create(C.byref(g), 100, 10, C.byref(p), 1, 0, 0, None, C.byref(h)) == dog.DOG_E_INVAL
    ids = (C.c_int * 2)(0, 0)
    assert dog.dog_create(C.byref(g), 100, 10, C.byref(p), 1, 0, 2, None, C.byref(h)) == dog.DOG_E_INVAL
    assert dog.dog_create(C.byref(g), 100, 10, C.byref(p), 1, 0, -1, ids, C.byref(h)) == dog.DOG_E_INVAL
    assert dog.dog_create(C.byref(g), 100, 10, C.byref(p), 1, dog.DOG_FLAG_DEBUG, 2, ids, C.byref(h)) == dog.DOG_E_INVAL
    assert dog.dog_step_sharded(None, None, 0.1, None) == dog.DOG_E_INVAL
    assert dog.dog_read_cells_sharded(None, None, None, None, None, None) == dog.DOG_E_INVAL
    assert dog.dog_set_bands(None, None) == dog.DOG_E_INVAL
    assert dog.dog_band_gather(None, None, None, None, None, 0, None, None, 0, None, None, None) == dog.DOG_E_INVAL
    assert dog.dog_step(None, None, 0.1, None) == dog.DOG_E_INVAL
    assert dog.dog_step_doppler(None, None, None, None, 0.1, None) == dog.DOG_E_INVAL
    assert dog.dog_step_exact(None, None, 0.1, None) == dog.DOG_E_INVAL
    assert dog.dog_step_exact_lik(None, None, None, None, 0.1, None) == dog.DOG_E_INVAL
    assert dog.dog_band_set_state(None, None, 0, 0, None, 0.0, 0) == dog.DOG_E_INVAL
    assert dog.dog_check_transforms(None) == dog.DOG_E_INVAL
    assert dog.dog_eval_cells(None, None, None, None, 0, None, None, None, 0, None, None, None, None) == dog.DOG_E_INVAL
    assert dog.dog_error_string(dog.DOG_E_MEAS)


def test_no_oracle_in_product():
    """The product path never imports or links the oracle, and ships no CPU fallback."""
    pkg = os.path.join(ROOT, "paper_1605_02406_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "dog_oracle" not in txt, f


def test_binding_fails_loudly_without_library(tmp_path):
    """With the CUDA library missing the product path refuses to import (no silent CPU fallback)."""
    import sys
    env = dict(os.environ, DOG_LIB=str(tmp_path / "missing" / "libdog.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_1605_02406_b200.dog"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "libdog.so not found" in r.stderr and "no fallback" in r.stderr
