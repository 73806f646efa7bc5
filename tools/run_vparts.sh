#!/bin/bash
# planner balance on one GPU: bench.py --virtual-parts G for cfg4 / cfg5 (slice times of vdmc_plan)
O=gpurun_out/${1:-vparts}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in cfg4 cfg5; do for G in ${VP_PARTS:-8 16}; do
  timeout 900 python bench.py --config $c --virtual-parts $G --steps 2 > $O/vparts_${c}_$G.json 2> $O/vparts_${c}_$G.err
done; done
