#!/bin/bash
# ncu --set full captures of k_enum (cfg4, cfg5) of the working tree + bench lines
O=gpurun_out/${1:-prof}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in ${PROF_CONFIGS:-cfg4 cfg5}; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_$c -f \
      python tools/profile_enum.py $c 4 1 > $O/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py $O/enum_$c.ncu-rep "$c k=4 k_enum" > $O/enum_${c}_summary.txt 2>&1
done
