#!/bin/bash
# One gpurun call: GPU parity suite, smoke, bench lines, ncu launch list + full captures of k_enum.
# usage (on the box): bash tools/gpu_check.sh [tag] [pytest-args...]
set -x
TAG=${1:-run}; shift
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf ${@:--x} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 python bench.py --config cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
for c in cfg4 cfg5; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_$c -f \
      python tools/profile_enum.py $c 4 1 > $O/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py $O/enum_$c.ncu-rep "$c k=4 k_enum" > $O/enum_${c}_summary.txt 2>&1
done
