#!/bin/bash
# GPU suite + default bench line of the working tree
O=gpurun_out/${1:-r02w}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 1500 python -m pytest tests -m gpu -x -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
