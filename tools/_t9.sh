O=gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_t9.log 2>&1; tail -2 $O/pytest_t9.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_t9.log 2>&1; tail -2 $O/smoke_t9.log
python bench.py > $O/bench_c3_t9.json 2> $O/bench_c3_t9.err; tail -c 400 $O/bench_c3_t9.json
bash tools/measure_configs.sh t9 c3f64 c2f64
