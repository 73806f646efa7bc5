#!/bin/bash
# k = 5 + layered parity, planner balance with the refit model, NEXT-2 / NEXT-3 bench lines + ncu
O=gpurun_out/${1:-r02e}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_k5.py tests/test_gpu_boundary.py tests/test_gpu_parity.py -q -rf -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --virtual-parts 8 --steps 1 > $O/vparts_cfg4.json 2> $O/vparts_cfg4.err
timeout 900 python bench.py --virtual-parts 8 --steps 1 --config cfg5 > $O/vparts_cfg5.json 2> $O/vparts_cfg5.err
timeout 900 python bench.py --config cfg3 --edges --no-cpu-baseline > $O/bench_edges_cfg3.json 2> $O/bench_edges_cfg3.err
timeout 900 python bench.py --config cfg5 --edges --no-cpu-baseline --steps 3 > $O/bench_edges_cfg5.json 2> $O/bench_edges_cfg5.err
timeout 900 python bench.py --config cfg2 --k 5 --no-cpu-baseline > $O/bench_k5_cfg2.json 2> $O/bench_k5_cfg2.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_edges -c 1 -o $O/edges_cfg3 -f \
    python tools/profile_enum.py cfg3 4 1 1.0 directed edges > $O/ncu_edges.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_layers -c 1 -o $O/layers_cfg2 -f \
    python tools/profile_enum.py cfg2 5 1 > $O/ncu_layers.log 2>&1
timeout 1500 python bench.py --config cfg4 --edges --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 1 > $O/bench_edges_cfg4.json 2> $O/bench_edges_cfg4.err
