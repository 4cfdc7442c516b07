#!/bin/bash
# One gpurun call: full ncu captures of C3r's face-ordered forward and
# single-face backward (the random-soup path), for their executed mixes.
# Usage: bash tools/measure_c3r.sh TAG
T=${1:-x}
O=gpurun_out
C="python bench.py --config c3r --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C > $O/plain_c3r_$T.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"(fwd|bwd)_f32_kernel" -s 2 -c 2 -o $O/ncu_c3r_$T $C > $O/ncu_c3r_$T.log 2>&1
tail -3 $O/ncu_c3r_$T.log; ls $O | tail -3
