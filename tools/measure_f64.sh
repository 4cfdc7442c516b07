#!/bin/bash
# One gpurun call: GPU parity of the trail kernels (f32 + f64), the f64
# default-precision lines (C2, C3) and an ncu capture of the f64 trail
# backward on the quarter-size c3s.  Usage: bash tools/measure_f64.sh TAG
T=${1:-x}
O=gpurun_out
python -m pytest tests/test_gpu_trail.py tests/test_gpu_f64_parity.py -q -p no:cacheprovider > $O/pytest_f64_$T.log 2>&1; tail -2 $O/pytest_f64_$T.log
bash tools/measure_configs.sh $T c2f64 c3f64
C="python bench.py --config c3s --precision f64 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C > $O/plain_f64_$T.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:bwd_f64_kernel -s 1 -c 1 -o $O/ncu_c3s_bwd64_$T $C > $O/ncu_bwd64_$T.log 2>&1
ls $O | tail -5
