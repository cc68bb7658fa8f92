"""Device-memory hygiene: libgis allocates from a
private pool per context, leaves the device's default pool untouched, and
gis_ctx_trim hands everything back."""

import pytest

pytestmark = pytest.mark.gpu


def _used():
    import torch

    free, total = torch.cuda.mem_get_info()
    return total - free


def test_trim_after_config5_run_releases_scratch():
    import gc

    import torch

    from paper_2202_06111_b200 import _device as D, run, trim
    from paper_2202_06111_b200.configs import config

    D.ctx()
    trim()
    base = _used()
    res = run(config(5))
    assert len(res.covering) == 7898713
    reserved = D.pool_reserved()
    assert reserved > (4 << 30), reserved  # config 5 grows several GB of scratch
    del res
    gc.collect()
    released = trim()
    assert released >= reserved - (64 << 20)
    assert D.pool_reserved() == 0
    assert _used() - base < (1 << 30), (_used() - base) / 2**30


def test_default_pool_release_threshold_untouched():
    import torch

    from paper_2202_06111_b200 import _device as D

    D.ctx()
    # the default pool's release threshold, read through the CUDA runtime
    # bindings (cuda-python): libgis must not have changed it from 0
    from cuda.bindings import runtime as R

    err, pool = R.cudaDeviceGetDefaultMemPool(torch.cuda.current_device())
    assert err == R.cudaError_t.cudaSuccess
    err, thr = R.cudaMemPoolGetAttribute(pool, R.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    assert err == R.cudaError_t.cudaSuccess
    assert int(thr) == 0
