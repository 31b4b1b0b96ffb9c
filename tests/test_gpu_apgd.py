"""GPU: the APGD dump / load (reference distances.py:149-177).

* byte-identical to the reference's own to_bytes on partially filled and
  complete stores (tests/golden/ref_apgd.npz, written by the reference);
* from_bytes of the reference's dumps restores dist, mark, counts and the
  filled total exactly as the reference's from_bytes;
* fp32 stores round-trip through the additive version 2;
* config 4 (128^2) and config 5 (256^2, a 32 GiB dump) stream through a
  checksum sink tile by tile -- never an N^2 host temporary -- and match the
  device array converted independently (torch).
"""

from __future__ import annotations

import io

import numpy as np
import pytest
import torch

from conftest import load_golden
from paper_2007_16076_b200.configs import CONFIGS, make_image

pytestmark = pytest.mark.gpu


def _cases(g):
    for i in range(int(g["n_cases"])):
        yield i, {k[len(f"c{i}_"):]: g[k] for k in g.files if k.startswith(f"c{i}_")}


def test_dump_bytes_equal_reference(gp):
    g = load_golden("ref_apgd.npz")
    for i, c in _cases(g):
        img = gp.Image(c["img"])
        graph = gp.GridGraph(img, gp.Metric.SUM)
        store = gp.DistanceArray(img.size)
        for r in c["roots"]:
            store.fill_from_tree(gp.build_tree(graph.propagate([int(r)]), int(r)))
        assert store.to_bytes() == c["partial"].tobytes(), i
        run = gp.run_strategy(img, gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
        assert run.distances.to_bytes() == c["full"].tobytes(), i


def test_load_reference_dumps(gp):
    g = load_golden("ref_apgd.npz")
    for i, c in _cases(g):
        blob = c["partial"].tobytes()
        st = gp.DistanceArray.from_bytes(blob)
        n = c["img"].size
        grid = np.frombuffer(blob, dtype="<u8", offset=9).reshape(n, n)
        mark = grid != gp.APGD_SENTINEL
        assert np.array_equal(st.mark, mark)
        assert np.array_equal(st.dist, np.where(mark, grid, 0).astype(np.int64) - (~mark))
        assert np.array_equal(st.point_filled_counts, c["partial_counts"])
        assert st.pairs_filled == int(c["partial_filled"])
        assert st.to_bytes() == blob
        st2 = gp.DistanceArray.read_apgd(io.BytesIO(c["full"].tobytes()))
        assert st2.is_complete and st2.to_bytes() == c["full"].tobytes()


def test_errors_match_reference(gp):
    g = load_golden("ref_apgd.npz")
    blob = g["c0_full"].tobytes()
    with pytest.raises(ValueError, match="bad magic"):
        gp.DistanceArray.from_bytes(b"XPGD" + blob[4:])
    with pytest.raises(ValueError, match="unsupported APGD version"):
        gp.DistanceArray.from_bytes(blob[:4] + bytes([7]) + blob[5:])
    with pytest.raises(ValueError, match="expected"):
        gp.DistanceArray.from_bytes(blob[:-8])
    bad = bytearray(blob)
    bad[9:17] = (1 << 30).to_bytes(8, "little")  # not representable in the fp32 store
    with pytest.raises(ValueError):
        gp.DistanceArray.from_bytes(bytes(bad))


def test_float_store_round_trip_version2(gp):
    img = np.random.default_rng(3).random((9, 11), dtype=np.float32)
    run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE)
    blob = run.distances.to_bytes()
    assert blob[4] == gp.APGD_VERSION_FLOAT
    grid = np.frombuffer(blob, dtype="<u8", offset=9).view("<f8").reshape(img.size, img.size)
    assert np.array_equal(grid.astype(np.float32), run.distances.dist)
    back = gp.DistanceArray.from_bytes(blob)
    assert np.array_equal(back.dist, run.distances.dist) and back.is_complete


class _Sink:
    """File-like checksum sink: wrapping u64 sums (plain and row-weighted)."""

    def __init__(self, n):
        self.n, self.head, self.rows, self.s1, self.s2 = n, b"", 0, np.uint64(0), np.uint64(0)
        self.peak = 0

    def write(self, b):
        b = memoryview(b)
        if not self.head:
            self.head = bytes(b)
            return len(b)
        self.peak = max(self.peak, b.nbytes)
        blk = np.frombuffer(b, dtype="<u8").reshape(-1, self.n)
        w = np.arange(self.rows + 1, self.rows + 1 + blk.shape[0], dtype=np.uint64)[:, None]
        with np.errstate(over="ignore"):
            self.s1 += blk.sum(dtype=np.uint64)
            self.s2 += (blk * w).sum(dtype=np.uint64)
        self.rows += blk.shape[0]
        return b.nbytes


def _expected(Dd, n, isf):
    s1, s2 = np.uint64(0), np.uint64(0)
    for r0 in range(0, n, 2048):
        blk = Dd[r0:r0 + 2048]
        blk = (blk.double().view(torch.int64) if isf else blk.to(torch.int64)).cpu().numpy().view(np.uint64)
        w = np.arange(r0 + 1, r0 + 1 + blk.shape[0], dtype=np.uint64)[:, None]
        with np.errstate(over="ignore"):
            s1 += blk.sum(dtype=np.uint64)
            s2 += (blk * w).sum(dtype=np.uint64)
    return s1, s2


@pytest.mark.parametrize("index", [4, 5])
def test_config_dump_streams(gp, index):
    spec = CONFIGS[index]
    run = gp.run_strategy(gp.Image(make_image(index)), gp.Metric.SUM, gp.StrategyKind.FILLING_RATE,
                          connectivity=spec.conn, force=True)
    sink = _Sink(spec.n)
    total = run.distances.write_apgd(sink)
    assert total == 9 + 8 * spec.n * spec.n and sink.rows == spec.n
    assert sink.head[4] == (gp.APGD_VERSION_FLOAT if spec.dtype == "f32" else gp.APGD_VERSION)
    assert sink.peak <= 64 << 20  # tiles, never an N^2 host buffer
    assert (sink.s1, sink.s2) == _expected(run.distances.dist_device(), spec.n, spec.dtype == "f32")
