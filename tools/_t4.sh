O=gpurun_out
python -m pytest tests/test_gpu_trail.py tests/test_trail.py -q -p no:cacheprovider > $O/pytest_trail4.log 2>&1; tail -2 $O/pytest_trail4.log
timeout 300 python tools/fwd_time.py --config c3 --bwd --path trails --reps 3
for v in k3 k4s2 k4m3 k4s8m3 k4s6m3; do WV_LIB_PATH=scratch/variants/$v/lib.so timeout 300 python tools/fwd_time.py --config c3 --bwd --path trails --reps 3; done
