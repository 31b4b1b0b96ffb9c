"""CPU: host-side logic of the drop-in package (no kernel launches)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2007_16076_b200 import configs
from paper_2007_16076_b200.grid import Image, Metric, edge_weight, neighbors, path_time
from paper_2007_16076_b200.propagation import PropagationResult, boundary_pixels, build_tree
from paper_2007_16076_b200.strategies import relative_difference, spiral_turns


def test_image_validation():
    with pytest.raises(ValueError):
        Image(np.array([[0, 1]]))
    with pytest.raises(ValueError):
        Image(np.array([[1, 256]]))
    with pytest.raises(ValueError):
        Image(np.array([1, 2]))
    with pytest.raises(ValueError):
        Image(np.array([[1.0, -0.5]]))
    img = Image(np.array([[1, 2], [3, 4]]))
    assert img.pixels.dtype == np.int64 and not img.pixels.flags.writeable
    f = Image(np.array([[0.0, 0.5]]))
    assert f.pixels.dtype == np.float32 and not f.is_integer


def test_neighbors_and_weights():
    assert neighbors((3, 3), 4) == [0, 1, 2, 3, 5, 6, 7, 8]
    assert neighbors((3, 3), 0) == [1, 3, 4]
    assert neighbors((3, 3), 4, connectivity=4) == [1, 3, 5, 7]
    img = Image.from_flat(3, 1, [1, 2, 3])
    assert edge_weight(img, Metric.SUM, 0, 1) == 6
    assert path_time(img, Metric.SUM, [0, 1, 2]) == 16
    assert edge_weight(Image.from_flat(2, 1, [5, 7]), Metric.L1, 0, 1) == 4
    assert edge_weight(Image.from_flat(2, 1, [5, 7]), Metric.MEAN, 0, 1) == 12


def test_build_tree_host():
    parent = np.array([-1, 0, 1, 0, 3], dtype=np.int64)
    res = PropagationResult((0,), np.array([0, 1, 2, 1, 2]), parent)
    tree = build_tree(res, 0)
    assert tree.children == [[1, 3], [2], [], [4], []]
    assert tree.leaves == [2, 4]
    with pytest.raises(ValueError):
        build_tree(res, 1)


def test_boundary_and_spiral():
    assert len(boundary_pixels((9, 9))) == 32
    assert boundary_pixels((3, 1)) == [0, 1, 2]
    assert spiral_turns(4, 4)[0] == [0, 1, 2, 3, 7, 11, 15, 14, 13, 12, 8, 4]
    assert [len(t) for t in spiral_turns(9, 9)] == [32, 24, 16, 8, 1]
    assert relative_difference(624, 468) == pytest.approx(25.0)


def test_config_generators_deterministic():
    for idx, spec in configs.CONFIGS.items():
        a, b = configs.make_image(idx), configs.make_image(idx)
        assert a.shape == spec.shape and np.array_equal(a, b)
        if spec.dtype == "u8":
            assert a.dtype == np.uint8 and a.min() >= 1
        else:
            assert a.dtype == np.float32 and a.min() >= 0 and a.max() <= 1


def test_gaussian_matches_scipy():
    nd = pytest.importorskip("scipy.ndimage")
    x = np.random.default_rng(3).standard_normal((30, 30))
    ref = nd.gaussian_filter(x, 2.0, mode="reflect", truncate=4.0)
    assert np.allclose(configs.gaussian_filter(x, 2.0), ref, atol=1e-12)


def test_partition_magic_division_is_exact():
    """commit.cu phase A: x / P == umulhi(x, ceil(2^42 / P)) >> 10 for x < 2^28 and P < 2^14
    (the unit chunk counts floor((p+1)T/P) - floor(pT/P) without 32-bit divisions)."""
    rng = np.random.default_rng(0)
    for P in (1025, 2049, 4736, 9472, 14208, 16383):
        M = ((1 << 42) + P - 1) // P
        assert M < (1 << 32)  # the constant fits 32 bits above 1024 partitions (capi.cu uses it only there)
        xs = np.concatenate([rng.integers(0, 1 << 28, 200_000, dtype=np.int64),
                             np.arange(0, 4 * P, dtype=np.int64), (1 << 28) - 1 - np.arange(0, 4 * P, dtype=np.int64),
                             (np.arange(1, 20_000, dtype=np.int64) * P) - 1, np.arange(1, 20_000, dtype=np.int64) * P])
        xs = xs[(xs >= 0) & (xs < (1 << 28))]
        q = ((xs.astype(object) * M) >> 32 >> 10).astype(np.int64)
        assert np.array_equal(q, xs // P), P
