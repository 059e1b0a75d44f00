# A/B helper: tests for the graph path, then C2/C4 bench lines per variant
set -x
O=gpurun_out/${TAG:-ab}; mkdir -p $O
python -m pytest tests/test_gpu_graphs.py -x -q > $O/tests.log 2>&1; tail -3 $O/tests.log
for v in "" "HARL_PAR_VALUE=1"; do
  env $v python bench.py --no-cpu-baseline > $O/c2_${v:-default}.json 2>>$O/err.log
done
python bench.py --config c4 --no-cpu-baseline > $O/c4.json 2>>$O/err.log
python bench.py --config c4 --no-cpu-baseline --steps 6 --warmup 2 > $O/c4_6.json 2>>$O/err.log
HARL_EAGER_CAPTURE=1 python bench.py --config c4 --no-cpu-baseline > $O/c4_eagercap.json 2>>$O/err.log
python profiles/segment_probe.py c2 > $O/seg_default.json 2>>$O/err.log
HARL_PAR_VALUE=1 python profiles/segment_probe.py c2 > $O/seg_par.json 2>>$O/err.log
