#!/bin/bash
# Round-2 final measurement of HEAD: smoke, bench lines, reference arm, ncu launch list, ncu captures of
# k_enum (cfg4, cfg5), planner balance (virtual parts), GPU suite.
O=gpurun_out/${1:-r02q}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --kind undirected --no-cpu-baseline > $O/bench_cfg4_und.json 2> $O/bench_cfg4_und.err
timeout 900 python bench.py --edges --config cfg3 --no-cpu-baseline > $O/bench_cfg3_edges.json 2> $O/bench_cfg3_edges.err
timeout 900 python bench.py --config cfg2 --k 5 --no-cpu-baseline > $O/bench_cfg2_k5.json 2> $O/bench_cfg2_k5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
for c in cfg4 cfg5; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_$c -f \
      python tools/profile_enum.py $c 4 1 > $O/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py $O/enum_$c.ncu-rep "$c k=4 k_enum" > $O/enum_${c}_summary.txt 2>&1
done
for c in cfg4 cfg5; do for G in 4 8 16; do
  timeout 900 python bench.py --config $c --virtual-parts $G --steps 2 > $O/vparts_${c}_$G.json 2> $O/vparts_${c}_$G.err
done; done
timeout 1500 python -m pytest tests -m gpu -x -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
