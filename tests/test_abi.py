"""CPU suite: the C-ABI libraries load and export every symbol the headers declare
(no compute calls: this container has no GPU)."""
import ctypes
import os
import re

import pytest

from paper_2501_13975_b200 import capi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(REPO, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|void|const char\*)\s+(ngs_\w+)\s*\(", src, re.M)))


def test_header_symbols_match_binding_list():
    assert sorted(capi.EXPORTED_SYMBOLS) == declared("ngs_b200.h")


@pytest.mark.parametrize("header", ["ngs_b200.h", "ngs_b200_profile.h", "ngs_b200_dist.h", "ngs_b200_ext.h"])
def test_product_library_exports_every_declared_symbol(header):
    assert os.path.exists(capi.PRODUCT_LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(capi.PRODUCT_LIB)
    for name in declared(header):
        assert hasattr(lib, name), name


def test_product_library_reports_backend_without_a_gpu():
    lib = capi.NgsLibrary(capi.PRODUCT_LIB)
    assert lib.backend == "cuda-sm_100a"
    assert lib.lib.ngs_abi_version() == 2
    r = lib.default_raster()
    assert (r.lambda_lp, r.alpha_cutoff, r.t_min, r.tiled) == (0.3, 1e-4, 1e-4, 1)   # rasterizer.hpp:25-31
    n = lib.default_newton()
    assert (n.mu_min, n.eig_floor_rel, n.step_cap_factor, n.scale_cap_factor, n.color_cap) == (1e-8, 5e-2, 1.0, 2.0, 1.0)
    t = lib.default_train()
    assert (list(t.order), t.knn, t.secondary_downsample, t.barrier_decay, t.barrier_floor) == \
        ([0, 1, 2, 3, 4], 3, 4, 0.5, 1e-6)                                              # trainer.hpp:58-77


def test_product_library_fails_loudly_without_a_device():
    lib = capi.NgsLibrary(capi.PRODUCT_LIB)
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(capi.NgsError):
        lib.context(0)


def test_reference_library_defaults_match_product():
    from refimpl import REF_LIB
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built")
    ref = capi.NgsLibrary(REF_LIB)
    prod = capi.NgsLibrary(capi.PRODUCT_LIB)
    for f in ("default_raster", "default_loss", "default_newton", "default_train"):
        a, b = getattr(ref, f)(), getattr(prod, f)()
        assert bytes(a) == bytes(b), f
