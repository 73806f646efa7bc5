O=gpurun_out/r01t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg5 -f \
    python tools/profile_enum.py cfg5 4 1 > $O/ncu_full5.log 2>&1
VDMC_PHASES=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg4_heavy -f \
    python tools/profile_enum.py cfg4 4 1 > $O/ncu_heavy.log 2>&1
