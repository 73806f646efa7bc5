#!/bin/bash
# round-2 measurement batch: new GPU tests, option A/B, bench lines, planner balance
O=gpurun_out/${1:-r02b}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_edges.py tests/test_gpu_hub.py -q -rf > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 600 python tools/ab_options.py cfg4 '{}' '{"star_block": 1023}' '{"star_block": 256}' > $O/ab_fold_cfg4.txt 2>&1
timeout 900 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --virtual-parts 8 --steps 1 > $O/vparts_cfg4.json 2> $O/vparts_cfg4.err
timeout 900 python bench.py --virtual-parts 8 --steps 1 --config cfg5 > $O/vparts_cfg5.json 2> $O/vparts_cfg5.err
