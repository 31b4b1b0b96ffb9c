"""Time the device extrema strategy on a config image (dev helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_16076_b200 as gp
from paper_2007_16076_b200.configs import CONFIGS, make_image

for idx in [int(a) for a in sys.argv[1:]] or [4]:
    spec = CONFIGS[idx]
    for rep in range(2):
        run = gp.run_strategy(gp.Image(make_image(idx)), gp.Metric.SUM, gp.StrategyKind.EXTREMA,
                              connectivity=spec.conn, force=True)
        st = run.stats
        print(f"cfg{idx} extrema rep{rep} P={run.trace.raw_count} dev_ms={st['ms_total']:.2f} "
              f"commit={st['ms_commit']:.2f} prop={st['ms_propagate']:.2f}", flush=True)
