#!/bin/bash
# quick GPU check of the working tree: build, parity subset, A/B of options on cfg4/cfg5
O=gpurun_out/${1:-quick}; shift; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_undirected.py tests/test_gpu_edges.py -x -q -rf > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
for c in ${AB_CONFIGS:-cfg4}; do timeout 600 python tools/ab_options.py $c "$@" >> $O/ab.txt 2>&1; done
