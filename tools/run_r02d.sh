#!/bin/bash
# memcheck, phase timings (profiling build), planner balance, A/B of light-path variants
O=gpurun_out/${1:-r02d}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "from paper_2201_11655_b200 import build as b; b.build_profiling()" >> $O/build.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_case.py > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
timeout 900 python tools/phase_probe.py cfg4 4 tasks > $O/phases_cfg4.txt 2>&1
timeout 900 python tools/phase_probe.py cfg5 4 quick > $O/phases_cfg5.txt 2>&1
timeout 900 python bench.py --virtual-parts 8 --steps 1 > $O/vparts_cfg4.json 2> $O/vparts_cfg4.err
timeout 900 python bench.py --virtual-parts 8 --steps 1 --config cfg5 > $O/vparts_cfg5.json 2> $O/vparts_cfg5.err
AB_CONFIGS="cfg4 cfg5" bash tools/ab.sh ${1:-r02d} default nolagather
