# Measurement of HEAD (one gpurun call): bench lines, reference arm, ncu launch list, ncu full captures.
# usage on the box: bash tools/measure_round.sh TAG   (outputs under gpurun_out/TAG)
O=gpurun_out/${1:-measure}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config cfg5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --kind undirected --no-cpu-baseline > $O/bench_cfg4_und.json 2> $O/bench_cfg4_und.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg4 -f \
    python tools/profile_enum.py cfg4 4 1 > $O/ncu_full4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_enum -c 1 -o $O/enum_cfg5 -f \
    python tools/profile_enum.py cfg5 4 1 > $O/ncu_full5.log 2>&1
