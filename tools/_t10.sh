timeout 300 python tools/fwd_time.py --config c3r --reps 3
for v in q0m3 q1m3 q1m4 q2m3; do WV_LIB_PATH=scratch/variants/$v/lib.so timeout 300 python tools/fwd_time.py --config c3r --reps 3; done
