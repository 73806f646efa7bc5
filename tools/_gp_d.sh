O=gpurun_out/r01d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
VDMC_TRACE=1 timeout 600 python tools/step_breakdown.py cfg5 4 3 > $O/trace_cfg5.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
