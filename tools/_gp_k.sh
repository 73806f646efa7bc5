O=gpurun_out/r01k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_undirected.py -x -q -k "small_fixtures or heavy_and_light or scaled or full_size or edge" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/phase_probe.py cfg4 4 > $O/phases_cfg4.txt 2>&1
timeout 600 python tools/phase_probe.py cfg5 4 > $O/phases_cfg5.txt 2>&1
