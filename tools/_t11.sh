timeout 300 python tools/fwd_time.py --config c3r --bwd --reps 3
for v in p1m5 p1m4 p0m4 p1m4s8; do WV_LIB_PATH=scratch/variants/$v/lib.so timeout 300 python tools/fwd_time.py --config c3r --bwd --reps 3; done
