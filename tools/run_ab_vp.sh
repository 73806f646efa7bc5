#!/bin/bash
# A/B of prebuilt variant libs: cfg4 phase timings + planner balance (virtual parts G = 8, 16)
O=gpurun_out/$1; shift; mkdir -p $O
for v in "$@"; do
  export VDMC_LIB=$PWD/paper_2201_11655_b200/lib/libvdmc_$v.so
  echo "== $v" >> $O/ab.txt
  timeout 600 python tools/phase_probe.py cfg4 4 quick >> $O/ab.txt 2>&1
  for G in 8 16; do
    timeout 900 python bench.py --config cfg4 --virtual-parts $G --steps 2 > $O/vparts_${v}_$G.json 2> $O/vparts_${v}_$G.err
    python -c "import json; d=json.loads(open('$O/vparts_${v}_$G.json').read().strip().splitlines()[-1]); print('G=$G max/mean %.3f ideal %.2f' % (d['max_over_mean'], d['ideal_speedup']), [round(x, 1) for x in d['slice_enum_ms']])" >> $O/ab.txt 2>&1
  done
done
