"""CPU: the multi-rank (replicas) aggregation of bench.py over gloo, world_size 2.

The path does not shard (replicas only); what runs across ranks
is the max-over-ranks timing and the whole-job throughput formula.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    local_ms = 100.0 * (rank + 1)  # rank 1 is the slow one
    total_ms, value = bench.aggregate(local_ms, pairs_per_image=1000, steps=4, world=world,
                                      dist=dist, device="cpu")
    q.put((rank, total_ms, value))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    for _, total_ms, value in res:
        assert total_ms == pytest.approx(200.0)  # max over ranks
        assert value == pytest.approx(2 * 1000 * 4 / 0.2)


def test_aggregation_single_rank():
    import bench

    total_ms, value = bench.aggregate(500.0, 10, 5, 1)
    assert total_ms == 500.0 and value == pytest.approx(100.0)


def test_committed_traffic_evidence_feeds_roofline():
    """bench.py's roofline.traffic comes from the committed ncu capture of the
    headline config; the commit kernels' bytes must be present and consistent."""
    import bench

    k, src = bench._traffic(5, ["k_commit", "k_commit_lb", "k_merge_sym"])
    assert src is not None and src.startswith("profiles/")
    assert k["launches"] > 0 and k["dram_bytes"] > 0
    assert abs(k["dram_bytes_per_launch"] * k["launches"] - k["dram_bytes"]) < 1e-6 * k["dram_bytes"]
    one, _ = bench._traffic(5, ["k_commit"])
    assert 0 < one["dram_bytes"] <= k["dram_bytes"]
    assert bench._traffic(999, ["k_commit"]) == (None, None)
    assert bench._traffic(5, ["no_such_kernel"]) == (None, None)


def test_both_arms_share_the_config_dict():
    """--impl reference builds its `config` with the same function and the same
    (golden) propagation counts as the repo arm, so the driver sees one config."""
    import bench
    from paper_2007_16076_b200.configs import CONFIGS

    P, P_adj, C = bench._golden_counts(5)
    assert (P, P_adj) == (52191, 52193) and C == 423501991006
    a = bench._config_dict(CONFIGS[5], P, P_adj, 1)
    assert a == bench._config_dict(CONFIGS[5], 52191, 52193, 1)
    assert a["workload"] == CONFIGS[5].name and a["pairs_per_image"] == CONFIGS[5].total_pairs


def test_cpu_baseline_sampler_runs_and_extrapolates():
    """bench._port_sample on the config-2 image (integer, 4096 pixels): the
    marginal-segment extrapolation returns a finite whole-image time bounded
    below by the sampled prefix, with the labels the JSON line carries."""
    import bench
    from paper_2007_16076_b200.configs import CONFIGS, make_image

    spec = CONFIGS[2]
    P, _, C = bench._golden_counts(2)
    assert C == 0 or C > 0  # the int goldens carry no visits (reference run)
    from oracle import oracle as O

    C = int(O.run(make_image(2), "filling-rate", nthreads=2)["visits"].sum())
    r = bench._port_sample(make_image(2), spec, P, C, 0.5, 2)
    assert r["kind"] == "port" and r["cores"] == 2 and r["commits_timed"] > 32
    assert r["ms_per_image"] / 1e3 > r["seconds"] * 0.5 and r["value"] > 0
    assert "extrapolated" in r["ms_per_image_kind"]


def test_reference_timing_script_replays_the_reference():
    """baseline/ref_timing.py runs the UNMODIFIED reference (when installed in
    baseline/_ref) over a replayed prefix of the committed cfg4 sequence."""
    import os

    import pytest

    import bench

    if not os.path.isdir(os.path.join(bench.ROOT, "baseline", "_ref", "geopairs")):
        pytest.skip("reference not installed in baseline/_ref")
    r = bench._ref_timing("replay", 4, 5, timeout=600)
    assert r.get("kind") == "reference", r
    assert r["commits"] == 5 and r["per_commit_ms"] > 0 and r["P"] == 13141
