O=gpurun_out/r01c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
VDMC_TRACE=1 timeout 600 python tools/step_breakdown.py cfg4 4 3 > $O/trace_cfg4.txt 2>&1
VDMC_TRACE=1 timeout 600 python tools/step_breakdown.py cfg5 4 3 > $O/trace_cfg5.txt 2>&1
