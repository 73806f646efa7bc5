O=gpurun_out/r01y; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in default noclob; do
  if [ $v = default ]; then unset VDMC_LIB; else export VDMC_LIB=$PWD/paper_2201_11655_b200/lib/libvdmc_$v.so; fi
  echo "== $v" >> $O/ab.txt
  timeout 600 python tools/phase_probe.py cfg4 4 quick >> $O/ab.txt 2>&1
  timeout 600 python tools/phase_probe.py cfg5 4 quick >> $O/ab.txt 2>&1
done
unset VDMC_LIB
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
