#!/bin/bash
# Measurement of HEAD: smoke, bench lines (cfg4 headline, cfg5, undirected, edge-level, k = 5,
# reference arm), ncu launch list, ncu --set full captures of k_enum (cfg4, cfg5), k_edges (cfg3)
# and k_layers (cfg2, k = 5).
O=gpurun_out/${1:-r02k}; mkdir -p $O
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
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_edges -c 1 -o $O/edges_cfg3 -f \
    python tools/profile_enum.py cfg3 4 1 1.0 directed edges > $O/ncu_full_edges.log 2>&1
python tools/ncu_summary.py $O/edges_cfg3.ncu-rep "cfg3 k=4 k_edges" > $O/edges_cfg3_summary.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_layers -c 1 -o $O/layers_cfg2 -f \
    python tools/profile_enum.py cfg2 5 1 > $O/ncu_full_layers.log 2>&1
python tools/ncu_summary.py $O/layers_cfg2.ncu-rep "cfg2 k=5 k_layers" > $O/layers_cfg2_summary.txt 2>&1
