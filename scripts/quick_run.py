"""Run one config through the public API and print timing stats (dev helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2007_16076_b200 as gp
from paper_2007_16076_b200.configs import CONFIGS, make_image

for idx in [int(a) for a in sys.argv[1:]] or [1, 2]:
    spec = CONFIGS[idx]
    img = make_image(idx)
    kind = gp.StrategyKind.FILLING_RATE if spec.strategy == "filling-rate" else gp.StrategyKind.NAIVE
    for rep in range(2):
        t0 = time.time()
        run = gp.run_strategy(gp.Image(img), gp.Metric.SUM, kind, connectivity=spec.conn, force=True)
        t1 = time.time()
        st = run.stats
        print(f"cfg{idx} rep{rep} wall={t1-t0:.3f}s P={run.trace.raw_count} dev_ms={st['ms_total']:.2f} "
              f"commit={st['ms_commit']:.2f} prop={st['ms_propagate']:.2f} setup={st['ms_setup']:.2f} "
              f"batches={st['batches']} props={st['propagations']} pairs/s={spec.total_pairs/(st['ms_total']/1e3):.3e}",
              flush=True)
