O=gpurun_out/r01s; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/phase_probe.py cfg4 4 quick > $O/phases_cfg4.txt 2>&1; timeout 600 python tools/phase_probe.py cfg5 4 quick > $O/phases_cfg5.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "heavy_and_light or scaled" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
