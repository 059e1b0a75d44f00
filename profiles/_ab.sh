O=gpurun_out/ab8; mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/tests.log 2>&1; tail -1 $O/tests.log
for i in 1 2; do
python bench.py --no-cpu-baseline > $O/new_$i.json 2>>$O/err.log
HARL_LIB_PATH=variants/old.so python bench.py --no-cpu-baseline > $O/old_$i.json 2>>$O/err.log
done
python bench.py --config c3 --no-cpu-baseline > $O/c3new.json 2>>$O/err.log
python bench.py --config c5 --no-cpu-baseline > $O/c5new.json 2>>$O/err.log
python profiles/phase_probe.py 16384 graph > $O/phase_new.txt 2>&1
