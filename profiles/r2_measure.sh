#!/bin/bash
# Round-2 measurement pass on one B200 (run from the repo root under gpurun).
# Outputs land in gpurun_out/r2/ ; summaries are copied into profiles/.
set -u
O=gpurun_out/r2
mkdir -p $O
T() { timeout "$@"; }
NCU=/usr/local/cuda/bin/ncu
[ -x $NCU ] || NCU=ncu

# 1. bench lines (no profiler attached)
T 900 python bench.py > $O/bench.json 2> $O/bench.err
T 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
# 2. MLP kernels alone at >= 64K rows (CUDA-event timer)
for c in "c3 65536" "c5 1048576"; do
  set -- $c
  T 300 python profiles/mlp_probe.py --config $1 --rows $2 --reps 5 --time > $O/mlp_$1_$2.json 2>&1
done
# 3. launch list of a short bench run (per-launch times, cold, serialised)
T 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline --no-extra > $O/launches_c2.log 2>&1
# 4. --set full of the tensor-core kernels at C3 64K and C5 1M
for c in "c3 65536" "c5 1048576"; do
  set -- $c
  T 900 $NCU --set full --clock-control none --import-source on \
    -k regex:"k_policy_tc|k_value_tc" --launch-skip 2 --launch-count 2 \
    -o $O/full_mlp_$1 -f python profiles/mlp_probe.py --config $1 --rows $2 --reps 3 \
    > $O/full_mlp_$1.log 2>&1
done
# 5. --set full of the C2 step kernels (traffic per launch)
T 1200 $NCU --set full --clock-control none --import-source on \
  -k regex:"k_sample_rows|k_gbt_finish|k_policy_tc|k_value_tc|k_ppo_rows|k_ppo_wgrad|k_ppo_adam" \
  --launch-skip 400 --launch-count 14 -o $O/full_c2 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/full_c2.log 2>&1
ls -la $O
