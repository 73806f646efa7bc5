O=gpurun_out/r01f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/phase_probe.py cfg4 4 > $O/phases_cfg4.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg5 -f \
    python tools/profile_enum.py cfg5 4 1 > $O/ncu_full5.log 2>&1
