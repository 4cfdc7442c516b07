#!/bin/bash
# One gpurun call with every round-end artefact: GPU tests, smoke, the C3
# line and its reference arm, the C3 launch list, full ncu captures of the
# C3 and C3r forwards (warp-row kernels), and the other configurations' lines.
# Usage: bash tools/measure_final.sh TAG
T=${1:-x}
O=gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_$T.log 2>&1; tail -1 $O/pytest_$T.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1; tail -1 $O/smoke_$T.log
python bench.py > $O/bench_c3_$T.json 2> $O/bench_c3_$T.err; tail -c 200 $O/bench_c3_$T.json
python bench.py --impl reference > $O/ref_c3_$T.json 2>&1; tail -c 150 $O/ref_c3_$T.json
C="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$C > $O/plain_$T.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_$T.csv $C > $O/ncu_launch_$T.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fwd_f32_kernel -s 1 -c 1 -o $O/ncu_c3_fwd_$T $C > $O/ncu_fwd_$T.log 2>&1
bash tools/measure_configs.sh $T c3r c2 c1 c4 c5
C="python bench.py --config c3r --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:fwd_f32_kernel -s 1 -c 1 -o $O/ncu_c3r_fwd_$T $C > $O/ncu_c3r_fwd_$T.log 2>&1
ls $O | grep $T
