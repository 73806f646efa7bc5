#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) + planner calibration (profiling build)
O=gpurun_out/${1:-r02c}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "from paper_2201_11655_b200 import build as b; b.build_profiling()" >> $O/build.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --leak-check none --print-limit 50 python tools/sanitize_case.py > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_case.py quick > $O/racecheck.txt 2>&1; echo "rc=$?" >> $O/racecheck.txt
timeout 1500 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_case.py quick > $O/synccheck.txt 2>&1; echo "rc=$?" >> $O/synccheck.txt
timeout 900 python tools/phase_probe.py cfg4 4 tasks > $O/phases_cfg4.txt 2>&1
timeout 900 python tools/phase_probe.py cfg5 4 quick > $O/phases_cfg5.txt 2>&1
