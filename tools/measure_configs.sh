#!/bin/bash
# One gpurun call: bench lines of the other BASELINE configs and of the f64
# default-precision path, timed regions >= 2 s (>= 10 NVML samples), into
# gpurun_out/line_<config>_<TAG>.json.  Usage: bash tools/measure_configs.sh TAG [configs...]
T=${1:-x}; shift
O=gpurun_out
run() { n=$1; shift; timeout 1500 python bench.py "$@" > $O/line_${n}_$T.json 2> $O/line_${n}_$T.err; echo "== $n rc=$?"; tail -c 250 $O/line_${n}_$T.json; echo; }
for c in ${@:-c3r c2 c1 c4 c2f64 c3f64 c5}; do
  case $c in
    c3r) run c3r --config c3r --steps 3 --warmup 3 ;;
    c2) run c2 --config c2 --steps 80 --warmup 5 ;;
    c1) run c1 --config c1 --steps 8000 --warmup 10 ;;
    c4) run c4 --config c4 --steps 40 --warmup 5 ;;
    c2f64) run c2f64 --config c2 --precision f64 --steps 5 --warmup 3 ;;
    c3f64) run c3f64 --config c3 --precision f64 --steps 1 --warmup 1 --cpu-nodes 8192 ;;
    c5) run c5 --config c5 --steps 1 --warmup 1 ;;
    ref_c4) run ref_c4 --impl reference --config c4 --steps 3 --warmup 1 ;;
    ref_c3r) run ref_c3r --impl reference --config c3r --steps 3 --warmup 1 ;;
  esac
done
