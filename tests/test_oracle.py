"""CPU: the oracle restatement pinned to the reference (golden vectors + KATs).

ref_small.npz and cfg2.npz/cfg4.npz were produced by running the unmodified
reference (tests/golden/make_golden.py); the known-answer tests restate the
reference's own unit tests (pkg/tests/test_propagation.py, test_distances.py).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import load_golden, small_cases
from paper_2007_16076_b200.configs import CONFIGS, make_image


def test_small_propagations_match_reference(ref_small, oracle):
    checked = 0
    for _, c in small_cases(ref_small):
        img, metric = c["img"], str(c["metric"])
        n = img.size
        for s in range(n):
            d, p = oracle.propagate(img, [s], metric=metric)
            assert np.array_equal(d, c["dist"][s])
            assert np.array_equal(p, c["parent"][s])
            checked += 1
    assert checked > 1000


def test_small_runs_match_reference(ref_small, oracle):
    for _, c in small_cases(ref_small):
        img, metric = c["img"], str(c["metric"])
        cen, dfc, ext = oracle.extrema(img, metric=metric)
        assert cen == int(c["centroid"])
        assert np.array_equal(dfc, c["dfc"]) and np.array_equal(ext, c["ext"])
        for tag, kind in (("naive", "naive"), ("fr", "filling-rate")):
            r = oracle.run(img, kind, metric=metric)
            assert np.array_equal(r["D"], c[tag + "_D"])
            assert np.array_equal(r["seq"], c[tag + "_seq"])
            assert r["adjusted"] == int(c[tag + "_adj"])


@pytest.mark.parametrize("index,stride", [(2, 1), (4, 1)])
def test_config_trees_match_reference_digests(oracle, index, stride):
    """The oracle's propagations on the config images against the reference's
    own (tests/golden/trees*.npz: cfg2 every source, cfg4 320 sources)."""
    g = load_golden(f"trees{index}.npz")
    img = make_image(index)

    def dig(a):
        return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).digest()[:16],
                             dtype=np.uint8)

    for i in range(0, len(g["src"]), stride):
        d, p = oracle.propagate(img, [int(g["src"][i])])
        assert np.array_equal(dig(d), g["dist_digest"][i]), int(g["src"][i])
        assert np.array_equal(dig(p), g["parent_digest"][i]), int(g["src"][i])


def test_cfg2_matches_reference_run(oracle):
    g = load_golden("cfg2.npz")
    r = oracle.run(make_image(2), "filling-rate", nthreads=4)
    assert r["raw"] == int(g["raw"]) and r["adjusted"] == int(g["adjusted"])
    assert np.array_equal(r["seq"], g["seq"])
    assert np.array_equal(r["new"], g["new"])
    assert hashlib.sha256(r["D"].astype("<i4").tobytes()).hexdigest() == str(g["d_sha256"])
    assert r["centroid"] == int(g["centroid"])


def test_cfg1_golden_is_oracle_output(oracle):
    g = load_golden("cfg1.npz")
    r = oracle.run(make_image(1), "naive")
    assert r["raw"] == int(g["raw"]) == 1023
    assert hashlib.sha256(r["D"].astype("<f4").tobytes()).hexdigest() == str(g["d_sha256"])


# ---- known-answer tests restated from the reference's unit tests ----
def test_kat_chain_distances(oracle):
    d, p = oracle.propagate(np.array([[1, 2, 3]]), [0])  # test_propagation.py:16-21
    assert d.tolist() == [0, 6, 16] and p.tolist() == [-1, 0, 1]


def test_kat_constant_image_chebyshev(oracle):
    f = 9  # test_propagation.py:23-30
    d, _ = oracle.propagate(np.full((5, 5), f), [12])
    cheb = np.array([[max(abs(r - 2), abs(c - 2)) for c in range(5)] for r in range(5)]).ravel()
    assert np.array_equal(d, 4 * f * cheb)


def test_kat_border_sources(oracle):
    border = [0, 1, 2, 3, 5, 6, 7, 8]  # test_propagation.py:32-37
    d, _ = oracle.propagate(np.full((3, 3), 7), border)
    assert d[4] == 28 and all(d[p] == 0 for p in border)


def test_kat_multi_source_is_min(oracle):
    rng = np.random.default_rng(33)  # test_propagation.py:63-73
    for _ in range(10):
        img = rng.integers(1, 256, (4, 5))
        srcs = list(rng.choice(20, size=int(rng.integers(2, 5)), replace=False))
        multi, _ = oracle.propagate(img, srcs)
        single = np.min([oracle.propagate(img, [s])[0] for s in srcs], axis=0)
        assert np.array_equal(multi, single)


def _store(n, isf=False):
    D = np.full((n, n), -1, dtype=np.float32 if isf else np.int64)
    np.fill_diagonal(D, 0)
    mark = np.eye(n, dtype=np.uint8)
    return D, mark, np.zeros(n, dtype=np.int64)


def test_kat_chain_fill(oracle):
    D, mark, cnt = _store(3)  # test_distances.py:63-71 and Fig. 1 anchor :73-77
    new, bad = oracle.fill_tree(np.array([-1, 0, 1]), np.array([0, 12, 20]), D, mark, cnt)
    assert new == 3 and bad == 0
    assert D[1, 2] == D[2, 1] == 8 and D[0, 2] == 20
    new, bad = oracle.fill_tree(np.array([-1, 0, 1]), np.array([0, 12, 20]), D, mark, cnt)
    assert new == 0 and bad == 0
    new, bad = oracle.fill_tree(np.array([-1, 0, 1]), np.array([0, 13, 20]), D, mark, cnt)
    assert bad > 0  # conflicting values (test_distances.py:100-104)


def test_kat_star_and_cycle(oracle):
    n = 6  # test_distances.py:79-83, 111-116
    D, mark, cnt = _store(n)
    new, _ = oracle.fill_tree(np.array([-1] + [0] * (n - 1)), np.array([0] + [4] * (n - 1)), D, mark, cnt)
    assert new == n - 1 and cnt[0] == n - 1
    D, mark, cnt = _store(3)
    new, _ = oracle.fill_tree(np.array([1, 0, -1]), np.array([0, 1, 2]), D, mark, cnt)
    assert new == -1


def test_fp32_mode_equals_int_mode_on_integer_images(oracle):
    rng = np.random.default_rng(5)
    for conn in (8, 4):
        img = rng.integers(1, 256, (9, 11))
        ri = oracle.run(img, "filling-rate", conn=conn)
        rf = oracle.run(img.astype(np.float32), "filling-rate", conn=conn)
        assert np.array_equal(ri["seq"], rf["seq"])
        assert np.array_equal(ri["D"].astype(np.float32), rf["D"])


def test_configs_golden_metadata():
    for idx, spec in CONFIGS.items():
        try:
            g = load_golden(f"cfg{idx}.npz")
        except pytest.skip.Exception:
            continue
        assert len(g["seq"]) == int(g["raw"])
        assert int(g["new"].sum()) == spec.total_pairs
