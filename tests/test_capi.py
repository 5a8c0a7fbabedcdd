"""The C-ABI library loads and exports every symbol include/tacho_b200.h declares."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "tacho_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b((?:tcg|tch)_[a-z_]+)\s*\(", text)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_1601_05871_b200 import _native
    lib = _native.load()
    declared = header_functions()
    assert len(declared) >= 30
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, f"declared but not exported: {missing}"


def test_python_binding_covers_the_header():
    from paper_1601_05871_b200 import _native
    bound = {name for name, _, _ in _native.SIGNATURES}
    assert set(header_functions()) <= bound


def test_struct_layouts_match_the_header():
    # field counts of the ctypes mirrors against the C declarations
    from paper_1601_05871_b200 import _native as N
    text = open(os.path.join(ROOT, "include", "tacho_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    for cname, py in (("tcg_problem", N.Problem), ("tcg_options", N.Options),
                      ("tcg_stats", N.Stats), ("tcg_plan_stats", N.PlanStats),
                      ("tcg_sym_stats", N.SymStats), ("tcg_solve_stats", N.SolveStats)):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + cname + ";", text, flags=re.S).group(1)
        decls = [d for d in body.split(";") if d.strip()]
        nfields = sum(len(d.split(",")) for d in decls)
        assert nfields == len(py._fields_), cname


def test_device_calls_fail_cleanly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1601_05871_b200 import _native as N
    lib = N.load()
    h = C.c_void_p()
    st = lib.tcg_create(0, C.byref(h))
    assert st == N.TCG_CUDA
    assert not h.value
    st = lib.tcg_sym_create(0, C.byref(h))
    assert st == N.TCG_CUDA
    assert not h.value


def test_plan_errors_map_to_reference_exceptions(T):
    a = T.generate("grid2d", 4, 4)
    an = T.analyze(a)
    bad = T.RangeList(an.ranges.bounds.copy())
    bad.bounds[-1] -= 1  # ranges no longer cover [0, n)
    with pytest.raises(ValueError, match="cover"):
        T.Plan(an.a_permuted, an.pattern, bad)
    with pytest.raises(ValueError):
        T.RangeList.from_ranges([(0, 3), (4, 16)])


DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin_with_reference_types")


@pytest.mark.skipif(not os.path.exists(DROPIN), reason="built only where /root/reference exists")
def test_cpp_dropin_compiles_against_reference_types_and_fails_cleanly_without_gpu():
    import subprocess

    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by tests/test_gpu_parity.py")
    r = subprocess.run([DROPIN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3, r.stdout + r.stderr
    assert "no device" in r.stdout
