"""ppipe_update_profiles_async: the upload happens inside the next enumerate, in
chunks overlapped with scoring (include/ppipe.h). Same bar as the main path:
bit-exact against the oracle / a fresh synchronous run."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import run_oracle
from tests.helpers import assert_same_result
from workloads import config3, config5

pytestmark = pytest.mark.gpu


def _scaled(w, f):
    return [np.minimum(m.lat_us.astype(np.uint64) * f // 4, 1 << 20).astype(np.uint32) for m in w.models]


def test_async_upload_replaces_the_loaded_values(oracle_built):
    w = config3()
    ctx = pp.load_profiles(_scaled(w, 7), [m.act_bytes for m in w.models], w.n_classes, w.batches, w.bw)
    try:
        pp.update_profiles_async(ctx, [m.lat_us for m in w.models], [m.act_bytes for m in w.models])
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert_same_result(pp.pareto(ctx), run_oracle(w), "config 3 after async upload")
        # the uploaded values stay: a second enumerate needs no new upload
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert_same_result(pp.pareto(ctx), run_oracle(w), "config 3 again")
    finally:
        pp.free(ctx)


def test_async_upload_chunks_config5_slice():
    w = config5(n_models=24)  # 4 chunks of 6 models
    ref = pp.run(w)
    ctx = pp.load_profiles(_scaled(w, 3), [m.act_bytes for m in w.models], w.n_classes, w.batches, w.bw)
    try:
        pp.update_profiles_async(ctx, [m.lat_us for m in w.models], [m.act_bytes for m in w.models])
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        g = pp.pareto(ctx)
        assert g.n_candidates == ref.n_candidates and g.n_feasible == ref.n_feasible
        assert np.array_equal(g.points.view(np.uint8), ref.points.view(np.uint8))
        assert np.array_equal(g.seg_offsets, ref.seg_offsets)
    finally:
        pp.free(ctx)


def test_async_upload_errors_surface_in_pareto(oracle_built):
    w = config3()
    lat = [m.lat_us.copy() for m in w.models]
    S = [m.act_bytes.copy() for m in w.models]
    bad = [x.copy() for x in lat]
    bad[11][3, :, 2] = (1 << 28) // bad[11].shape[1] + 1
    ctx = pp.load_workload(w)
    try:
        pp.update_profiles_async(ctx, bad, S)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        with pytest.raises(pp.PPipeError) as e:
            pp.pareto(ctx)
        assert e.value.code == -2
        assert f"model 11 class 3 batch {int(w.batches[2])}: whole-model latency" in str(e.value)
        with pytest.raises(pp.PPipeError) as e2:
            pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert e2.value.code == -6
        # a synchronous update after a pending asynchronous one wins
        pp.update_profiles_async(ctx, bad, S)
        pp.update_profiles(ctx, lat, S)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert_same_result(pp.pareto(ctx), run_oracle(w), "recovered")
    finally:
        pp.free(ctx)


@pytest.mark.parametrize("value", [0xFFFFFFFF, 0x80000000, (1 << 28)])
def test_async_upload_of_wrapping_latencies_fails_cleanly(oracle_built, value):
    """Values that would wrap an int32 prefix sum (UINT32_MAX markers, 2^31) are packed
    and scored before the device validation result is read: the pack saturates, so
    pareto reports ERANGE (not an illegal address) and the context recovers."""
    w = config3()
    lat = [m.lat_us.copy() for m in w.models]
    S = [m.act_bytes.copy() for m in w.models]
    bad = [x.copy() for x in lat]
    bad[5][1, :, :] = np.uint32(value)
    bad[6][0, 0, 0] = np.uint32(value)
    ctx = pp.load_workload(w)
    try:
        pp.update_profiles_async(ctx, bad, S)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        with pytest.raises(pp.PPipeError) as e:
            pp.pareto(ctx)
        assert e.value.code == -2 and "model 5 class 1 batch" in str(e.value)
        pp.update_profiles(ctx, lat, S)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert_same_result(pp.pareto(ctx), run_oracle(w), "recovered after wrapping values")
    finally:
        pp.free(ctx)


def test_async_upload_same_buffers_new_contents(oracle_built):
    """A serving loop re-uploads the same (pinned) arrays with new contents: the cached
    descriptors must point at the live buffers, and slices of one buffer (merged copies)
    must land per model."""
    w = config3()
    lat_all = np.zeros(sum(m.lat_us.size for m in w.models), np.uint32)
    S_all = np.zeros(sum(m.act_bytes.size for m in w.models), np.uint64)
    lat, S, ol, os_ = [], [], 0, 0
    for m in w.models:
        lat.append(lat_all[ol:ol + m.lat_us.size].reshape(m.lat_us.shape))
        S.append(S_all[os_:os_ + m.act_bytes.size].reshape(m.act_bytes.shape))
        ol += m.lat_us.size
        os_ += m.act_bytes.size
    for a, m in zip(lat, _scaled(w, 7)):
        a[...] = m
    for a, m in zip(S, w.models):
        a[...] = m.act_bytes
    ctx = pp.load_profiles(lat, S, w.n_classes, w.batches, w.bw)
    try:
        pp.update_profiles_async(ctx, lat, S)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        g7 = pp.pareto(ctx)
        for a, m in zip(lat, w.models):  # new contents, same array objects
            a[...] = m.lat_us
        pp.update_profiles_async(ctx, lat, S)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert_same_result(pp.pareto(ctx), run_oracle(w), "config 3, same buffers with new contents")
        assert g7.n_points != 0
    finally:
        pp.free(ctx)
