O=gpurun_out/r01j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
VDMC_PHASES=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg4_heavy -f python tools/profile_enum.py cfg4 4 1 > $O/ncu_heavy.log 2>&1
VDMC_PHASES=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg4_light -f python tools/profile_enum.py cfg4 4 1 > $O/ncu_light.log 2>&1
