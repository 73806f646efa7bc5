#!/bin/bash
# Confirmation of HEAD's bench lines with the refreshed ncu counters + an ncu capture of the undirected kernel
O=gpurun_out/${1:-r02u}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg4_und -f \
    python tools/profile_enum.py cfg4 4 1 1.0 undirected > $O/ncu_full_und.log 2>&1
python tools/ncu_summary.py $O/enum_cfg4_und.ncu-rep "cfg4 k=4 undirected k_enum" > $O/enum_cfg4_und_summary.txt 2>&1
