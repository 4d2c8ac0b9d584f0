"""The host-core implementation of the paper's enumeration (cpu_method/) against the
brute-force oracle: identical unit counts on every ray, forward values to fp64 rounding."""
import numpy as np
import pytest

import cpu_method
import oracle
import workloads
from oracle import geometry as G

import helpers as H


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_cpu_method_matches_oracle(idx):
    c = H.small_config(idx)
    ids = workloads.sample_rays(c, 1500, seed=40 + idx)
    p, th = G.rays(c, ids)
    img = workloads.make_image(c).numpy().reshape(-1)
    val, cnt = cpu_method.forward(c, img, p, th, with_counts=True)
    rp, cols, lens = oracle.rows(c, p, th, mode=1)
    assert np.array_equal(cnt, np.diff(rp))
    ref = oracle.forward(c, img, p, th, mode=1)
    assert np.max(np.abs(val - ref)) <= 1e-11 * max(1.0, np.max(np.abs(ref)))


def test_cpu_method_constructed_edge_rays():
    """The 32 constructed edge / diagonal rays on 64^2: closed-form row sizes."""
    for g, expect in H.constructed_plans():
        ids = np.array(sorted(expect))
        p, th = G.rays(g, ids)
        img = np.ones(64 * 64, dtype=np.float32)
        _, cnt = cpu_method.forward(g, img, p, th, with_counts=True)
        assert cnt.tolist() == [expect[i] for i in ids.tolist()]
