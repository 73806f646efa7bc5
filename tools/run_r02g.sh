#!/bin/bash
# Re-entry check of HEAD: full GPU suite, smoke, u32/u64 accumulator A/B, bench lines, ncu launch list + k_enum captures
O=gpurun_out/${1:-r02g}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg5 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 python tools/ab_options.py cfg4 "{}" "{\"star_block\": 1023}" > $O/ab_closed_cfg4.txt 2>&1
timeout 600 python tools/ab_options.py cfg5 '{}' '{"acc64": 1}' > $O/ab_acc_cfg5.txt 2>&1
timeout 600 python tools/profile_enum.py cfg2 5 2 > $O/k5_cfg2.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=25 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
for c in cfg4 cfg5; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_$c -f \
      python tools/profile_enum.py $c 4 1 > $O/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py $O/enum_$c.ncu-rep "$c k=4 k_enum" > $O/enum_${c}_summary.txt 2>&1
done
