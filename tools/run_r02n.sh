#!/bin/bash
# planner refit data: slice times of vdmc_plan (bench.py --virtual-parts G) and phase totals
O=gpurun_out/${1:-r02n}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in cfg4 cfg5; do
  timeout 600 python tools/phase_probe.py $c 4 quick > $O/phases_$c.txt 2>&1
  for G in ${VP_PARTS:-4 8 16}; do
    timeout 900 python bench.py --config $c --virtual-parts $G --steps 2 > $O/vparts_${c}_$G.json 2> $O/vparts_${c}_$G.err
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
