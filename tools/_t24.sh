for v in default k3m5 k3m4 k3m5s4 default; do L=""; [ $v != default ] && L="WV_LIB_PATH=scratch/variants/$v/lib.so"; env $L timeout 300 python tools/fwd_time.py --config c3 --bwd --reps 3; done
