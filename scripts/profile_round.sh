#!/bin/bash
# Round profile capture on one B200 (run under gpurun from the repo root).
#   scripts/profile_round.sh r01 [config]
# Every ncu command runs only after the same program exited 0 without ncu.
# Outputs land in gpurun_out/<tag>_*; summaries are copied into profiles/ by hand.
set -u
TAG=${1:-r02}
CFG=${2:-5}
O=gpurun_out
mkdir -p $O
NCU="ncu --clock-control none"
echo "== plain runs"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-others --config $CFG > $O/${TAG}_bench_plain.json 2> $O/${TAG}_bench_plain.err || exit 1
timeout 300 python scripts/one_run.py $CFG > $O/${TAG}_one_run.log 2>&1 || exit 1
echo "== launch list"
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file $O/${TAG}_cfg${CFG}_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-others --config $CFG > $O/${TAG}_ncu_launches.log 2>&1
echo "launches exit $?"
echo "== per-kernel DRAM traffic of one image"
timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file $O/${TAG}_cfg${CFG}_traffic.csv python scripts/one_run.py $CFG > $O/${TAG}_ncu_traffic.log 2>&1
echo "traffic exit $?"
echo "== full captures"
# tree-mode commit kernel (mangled name ...ELi0E) and the batched list-mode kernel k_commit_lb
timeout 900 $NCU --set full --import-source on --kernel-name-base mangled -k regex:k_commitILi4ELi1024ELi1ELi0E --launch-skip 20 --launch-count 1 \
  -o $O/${TAG}_cfg${CFG}_k_commit_tree -f python scripts/one_run.py $CFG > $O/${TAG}_ncu_commit_tree.log 2>&1
echo "commit tree exit $?"
timeout 900 $NCU --set full --import-source on -k regex:k_commit_lb --launch-skip 100 --launch-count 1 \
  -o $O/${TAG}_cfg${CFG}_k_commit_list -f python scripts/one_run.py $CFG > $O/${TAG}_ncu_commit_list.log 2>&1
echo "commit list exit $?"
GP_PIPELINE=0 timeout 900 $NCU --set full --import-source on -k regex:k_propagate --launch-skip 40 --launch-count 1 \
  -o $O/${TAG}_cfg${CFG}_k_propagate -f python scripts/one_run.py $CFG > $O/${TAG}_ncu_prop.log 2>&1
echo "propagate exit $?"
ls -la $O
