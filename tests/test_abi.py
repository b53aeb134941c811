"""CPU: the C-ABI library loads, exports every symbol include/fppm_gpu.h
declares, and its host-side numerics (critical values, radius schedule) match
the reference bit for bit.  No GPU compute is invoked here."""
import json
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fppm_gpu.h")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fppm_gpu_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("fppm_gpu_create", "fppm_gpu_destroy", "fppm_gpu_set_photons",
              "fppm_gpu_build_grid", "fppm_gpu_query_ball", "fppm_gpu_gather_test",
              "fppm_gpu_iterate", "fppm_gpu_end_iteration", "fppm_gpu_accumulate"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2504_04411_b200 import _native
    lib = _native.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding covers the whole ABI
    assert set(declared_symbols()) <= set(_native.EXPORTED)


def test_abi_version_and_status_strings():
    from paper_2504_04411_b200 import _native
    lib = _native.lib()
    assert lib.fppm_gpu_abi_version() == 1
    assert lib.fppm_gpu_status_string(0) == b"ok"
    assert lib.fppm_gpu_status_string(2) == b"domain error"


def test_host_critical_values_match_reference():
    from paper_2504_04411_b200 import chi2_quantile, f_quantile
    for c in GOLDEN["f_quantile"]:
        assert f_quantile(c["p"], c["d1"], c["d2"]) == float.fromhex(c["value"]), c
    for c in GOLDEN["chi2_quantile"]:
        assert chi2_quantile(c["p"], c["df"]) == float.fromhex(c["value"]), c


def test_host_schedule_matches_reference():
    from paper_2504_04411_b200 import schedule_radius
    for c in GOLDEN["schedule_radius"]:
        assert schedule_radius(c["base"], c["alpha"], c["i"]) == float.fromhex(c["value"])


def test_invalid_quantile_arguments_raise():
    from paper_2504_04411_b200 import InvalidArgument, f_quantile
    with pytest.raises(InvalidArgument):
        f_quantile(1.0, 2.0, 2.0)
    with pytest.raises(InvalidArgument):
        f_quantile(0.5, 0.0, 2.0)


def test_context_without_gpu_fails_loudly():
    """No CPU fallback: creating a context needs an sm_100 device."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2504_04411_b200 import FppmContext, NoDeviceError
    with pytest.raises(NoDeviceError):
        FppmContext(initial_radius=0.02, samples_per_iteration=16, max_hitpoints=4, max_photons=16)


def test_config_validation_matches_gatherregion_ctor():
    """gather.cpp:41-50 checks run before any device probing."""
    from paper_2504_04411_b200 import FppmContext, InvalidArgument
    bad = [dict(initial_radius=0.0), dict(k=1.5), dict(alpha=0.3), dict(r_min_base=2.0),
           dict(n_annuli=1, n_sectors=1)]
    for over in bad:
        kw = dict(initial_radius=1.0, samples_per_iteration=10, r_min_base=0.001)
        kw.update(over)
        with pytest.raises(InvalidArgument):
            FppmContext(**kw)
