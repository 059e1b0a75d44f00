#!/bin/bash
# Round-2 population sweep (C5 1K -> 1M) and the C1/C3 lines, one B200.
O=gpurun_out/r2_sweep
mkdir -p $O
for P in 1024 4096 16384 65536 262144 1048576; do
  timeout 600 python bench.py --config c5 --population $P --steps 5 --warmup 3 \
    --no-cpu-baseline --no-extra > $O/c5_$P.json 2> $O/c5_$P.err
done
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > $O/c1.json 2> $O/c1.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-extra > $O/c3.json 2> $O/c3.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 > $O/c4.json 2> $O/c4.err
timeout 900 python bench.py --config c4 --impl reference --steps 2 --warmup 0 > $O/c4_reference.json 2> $O/c4_reference.err
ls -la $O
