#!/bin/bash
# GPU check of the working tree: build, A/B of variant libs (cfg4, cfg5), then the GPU suite.
O=gpurun_out/${1:-r02h}; shift; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
AB_CONFIGS="cfg4 cfg5" bash tools/ab.sh ${O#gpurun_out/} "$@"
timeout 1500 python -m pytest tests -m gpu -x -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
