O=gpurun_out
for v in default m3 u2 m3u2; do L=""; [ $v != default ] && L="WV_LIB_PATH=scratch/variants/$v/lib.so"; env $L timeout 600 python tools/fwd_time.py --config c3s --bwd --precision f64 --reps 3; done
python bench.py --steps 3 --warmup 3 > $O/bench_c3_t8.json 2> $O/bench_c3_t8.err; python -c "
import json; d=json.loads(open('$O/bench_c3_t8.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e'])"
