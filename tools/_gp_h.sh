O=gpurun_out/r01h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_fixtures or heavy_and_light or scaled or full_size" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/phase_probe.py cfg5 4 > $O/phases_cfg5.txt 2>&1
timeout 600 python tools/phase_probe.py cfg4 4 > $O/phases_cfg4.txt 2>&1
for ph in 1 2; do VDMC_PHASES=$ph timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_red.sum,smsp__inst_executed.sum --clock-control none -k regex:k_enum -c 1 python tools/profile_enum.py cfg4 4 1 > $O/ncu_phase$ph.txt 2>&1; done
