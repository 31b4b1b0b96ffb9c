"""Experiment layer (reference harness.py): test-image families on the CPU,
the experiment runner and its byte-identical CSV reports on the GPU, and the
reference's aggregate known answers (mean filling-rate propagation counts)."""

from __future__ import annotations

from statistics import fmean

import numpy as np
import pytest

from conftest import load_golden


def test_generated_images_equal_the_references():
    from paper_2007_16076_b200.harness import GeneratorKind, generate_image, hairpin_corridor_mask

    g = load_golden("ref_harness.npz")
    sizes = [(25, 25), (12, 9), (7, 16), (31, 20)]
    for kind in GeneratorKind:
        for si, size in enumerate(sizes):
            for seed in (0, 3, 19):
                img = generate_image(kind, size, seed)
                assert np.array_equal(img.pixels, g[f"img_{kind.value}_{si}_{seed}"]), (kind, size, seed)
    for si, (w, h) in enumerate(sizes):
        assert np.array_equal(hairpin_corridor_mask(w, h), g[f"mask_{si}"])
    with pytest.raises(ValueError):
        generate_image(GeneratorKind.RANDOM, (1, 1))


@pytest.mark.gpu
def test_experiment_csv_reports_are_byte_identical(gp):
    g = load_golden("ref_harness.npz")
    images = [(f"{k.value}8", gp.generate_image(k, (8, 7), 5)) for k in gp.GeneratorKind]
    kinds = [gp.StrategyKind.NAIVE, gp.StrategyKind.SPIRAL, gp.StrategyKind.SPIRAL_REPULSION,
             gp.StrategyKind.EXTREMA, gp.StrategyKind.FILLING_RATE]
    rep = gp.run_experiment(images, [gp.Metric.SUM, gp.Metric.MEAN], kinds, [0, 1], verify=True)
    assert gp.write_trace_csv(rep.records) == g["trace_csv"].tobytes()
    assert gp.write_report_csv(rep) == g["report_csv"].tobytes()


@pytest.mark.gpu
def test_filling_rate_family_means(gp):
    """The reference's aggregate pins (conftest.py:77-103, test_output.txt:224):
    mean filling-rate raw counts 286.75 / 387.4 / 465.9 on 25x25 bumps /
    hairpin / random, seeds 0..19."""
    want = {"bumps": 286.75, "hairpin": 387.4, "random": 465.9}
    for kind in gp.GeneratorKind:
        raws = [gp.run_strategy(gp.generate_image(kind, (25, 25), seed=k), gp.Metric.SUM,
                                gp.StrategyKind.FILLING_RATE, seed=k).trace.raw_count for k in range(20)]
        assert fmean(raws) == pytest.approx(want[kind.value], abs=1e-9), kind
