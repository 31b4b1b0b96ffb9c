"""One run of config C through the public API (profiling helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_16076_b200 as gp
from paper_2007_16076_b200.configs import CONFIGS, make_image

idx = int(sys.argv[1])
spec = CONFIGS[idx]
kind = gp.StrategyKind.FILLING_RATE if spec.strategy == "filling-rate" else gp.StrategyKind.NAIVE
run = gp.run_strategy(gp.Image(make_image(idx)), gp.Metric.SUM, kind, connectivity=spec.conn, force=True)
print(f"cfg{idx} P={run.trace.raw_count} stats={run.stats}")
