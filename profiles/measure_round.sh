set -x
mkdir -p gpurun_out/${TAG:-v6}
python bench.py > gpurun_out/${TAG:-v6}/bench.json 2> gpurun_out/${TAG:-v6}/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG:-v6}/bench_reference.json 2> gpurun_out/${TAG:-v6}/ref.err
for P in 1024 4096 16384 65536 262144 1048576; do python bench.py --config c5 --population $P --no-cpu-baseline > gpurun_out/${TAG:-v6}/sweep_c5_$P.json 2>>gpurun_out/${TAG:-v6}/sweep.err; done
python bench.py --config c1 --no-cpu-baseline > gpurun_out/${TAG:-v6}/c1.json 2>>gpurun_out/${TAG:-v6}/sweep.err
python bench.py --config c3 --no-cpu-baseline > gpurun_out/${TAG:-v6}/c3.json 2>>gpurun_out/${TAG:-v6}/sweep.err
python bench.py --config c4 --no-cpu-baseline > gpurun_out/${TAG:-v6}/c4.json 2>>gpurun_out/${TAG:-v6}/sweep.err
python profiles/segment_probe.py c2 > gpurun_out/${TAG:-v6}/segments.json 2>>gpurun_out/${TAG:-v6}/sweep.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG:-v6}/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG:-v6}/ncu_bench.log 2>&1

ncu --set full --clock-control none --import-source on -k 'regex:k_sample_rows|k_gbt_finish|k_value_tc|k_policy_tc64' --launch-skip 150 --launch-count 4 -o gpurun_out/${TAG:-v6}/full python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG:-v6}/ncu_full.log 2>&1
