#!/bin/bash
# One gpurun call: GPU tests, the headline C3 line (our arm + reference arm),
# the launch list of the same command and a full ncu capture of the strip
# forward (C3), into gpurun_out/.  Usage: bash tools/measure_c3.sh TAG
T=${1:-x}
O=gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_$T.log 2>&1; tail -2 $O/pytest_$T.log
python bench.py --steps 5 --warmup 3 > $O/bench_c3_$T.json 2> $O/bench_c3_$T.err; tail -c 300 $O/bench_c3_$T.json
python bench.py --impl reference --steps 5 --warmup 3 > $O/ref_c3_$T.json 2>&1; tail -c 200 $O/ref_c3_$T.json
C="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$C > $O/plain_$T.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_$T.csv $C > $O/ncu_launch_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bwd_f32_kernel -s 0 -c 1 -o $O/ncu_c3_bwd_$T $C > $O/ncu_bwd_$T.log 2>&1
ls $O | tail -20
