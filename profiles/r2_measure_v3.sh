#!/bin/bash
# Round-2 measurement pass on one B200 (repo root, under gpurun):
# bench lines, launch list and --set full capture of the C2 step kernels,
# --set full of the MLP kernels at C3 64 K / C5 1 M, the population sweep
# and the probes.  Outputs in gpurun_out/${TAG:-r2v3}/.
set -u
O=gpurun_out/${TAG:-r2v3}
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
EPI='regex:k_(mlp_f16|sample|gbt|ppo|featurize|gather|init|finish)'
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python profiles/segment_probe.py c2 > $O/segments.json 2>/dev/null
python profiles/host_probe.py > $O/host.json 2>/dev/null
python profiles/e2e_probe.py > $O/e2e.txt 2>&1
python profiles/overlap_probe.py 8192 > $O/overlap_8k.json 2>&1
for c in "c3 65536" "c5 1048576"; do
  set -- $c
  timeout 300 python profiles/mlp_probe.py --config $1 --rows $2 --reps 5 --time --phases > $O/mlp_$1_$2.json 2>&1
done
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k "$EPI" -c 3000 --csv \
  --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 \
  --no-cpu-baseline --no-extra > $O/launches_c2.log 2>&1
timeout 1200 $NCU --set full --clock-control none --import-source on \
  -k regex:"k_sample_rows|k_gbt_finish|k_mlp_f16|k_ppo_rows|k_ppo_wgrad|k_ppo_adam" \
  --launch-skip 400 --launch-count 14 -o $O/full_c2 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/full_c2.log 2>&1
$NCU -i $O/full_c2.ncu-rep --page raw --csv > $O/full_c2.raw.csv 2>/dev/null
rm -f $O/full_c2.ncu-rep
for c in "c3 65536" "c5 1048576"; do
  set -- $c
  timeout 900 $NCU --set full --clock-control none --import-source on \
    -k regex:"k_mlp_f16" --launch-skip 2 --launch-count 2 \
    -o $O/full_mlp_$1 -f python profiles/mlp_probe.py --config $1 --rows $2 --reps 2 \
    > $O/full_mlp_$1.log 2>&1
  $NCU -i $O/full_mlp_$1.ncu-rep --page raw --csv > $O/full_mlp_$1.raw.csv 2>/dev/null
  rm -f $O/full_mlp_$1.ncu-rep
done
for P in 1024 16384 65536 262144 1048576; do
  timeout 600 python bench.py --config c5 --population $P --steps 5 --warmup 3 \
    --no-cpu-baseline --no-extra > $O/c5_$P.json 2> $O/c5_$P.err
done
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > $O/c1.json 2> $O/c1.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-extra > $O/c3.json 2> $O/c3.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 > $O/c4.json 2> $O/c4.err
ls -la $O
