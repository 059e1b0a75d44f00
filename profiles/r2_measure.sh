#!/bin/bash
# Round-2 measurement pass on one B200 (run from the repo root under gpurun).
# Outputs land in gpurun_out/r2/ ; summaries are copied into profiles/.
set -u
O=gpurun_out/r2
mkdir -p $O
T() { timeout "$@"; }
NCU=/usr/local/cuda/bin/ncu
[ -x $NCU ] || NCU=ncu
EPI='regex:k_(mlp_f16|policy|sample|value|gbt|ppo|featurize|gather|init|finish)'

# 1. bench lines (no profiler attached)
T 900 python bench.py > $O/bench.json 2> $O/bench.err
T 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
# 2. tensor-core MLPs and the sampler alone at >= 64K rows (CUDA-event timer)
for c in "c3 65536" "c5 1048576"; do
  set -- $c
  T 300 python profiles/mlp_probe.py --config $1 --rows $2 --reps 5 --time --phases > $O/mlp_$1_$2.json 2>&1
done
# 3. launch list of a short bench run, episode kernels only (per-launch
#    times, cold, serialised)
T 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k "$EPI" -c 3000 --csv \
  --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline --no-extra > $O/launches_c2.log 2>&1
# 4. --set full of the tensor-core kernels and the sampler at C3 64K and C5 1M
for c in "c3 65536" "c5 1048576"; do
  set -- $c
  T 900 $NCU --set full --clock-control none --import-source on \
    -k regex:"k_mlp_f16|k_sample_rows|k_featurize2" --launch-skip 3 --launch-count 4 \
    -o $O/full_mlp_$1 -f python profiles/mlp_probe.py --config $1 --rows $2 --reps 3 \
    > $O/full_mlp_$1.log 2>&1
done
# 5. --set full of the C2 step kernels (traffic per launch)
T 1200 $NCU --set full --clock-control none --import-source on \
  -k regex:"k_sample_rows|k_gbt_finish|k_mlp_f16|k_ppo_rows|k_ppo_wgrad|k_ppo_adam" \
  --launch-skip 400 --launch-count 14 -o $O/full_c2 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/full_c2.log 2>&1
# keep the returned directory small (gpurun copies back <= 64 MiB): the
# captures are exported to CSV here and the .ncu-rep files dropped
for f in $O/*.ncu-rep; do
  b=${f%.ncu-rep}
  $NCU -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  $NCU -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $f
done
ls -la $O
