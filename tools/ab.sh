O=gpurun_out/$1; shift; mkdir -p $O
for v in "$@"; do
  if [ $v = default ]; then unset VDMC_LIB; else export VDMC_LIB=$PWD/paper_2201_11655_b200/lib/libvdmc_$v.so; fi
  echo "== $v" >> $O/ab.txt
  timeout 600 python tools/phase_probe.py cfg4 4 quick >> $O/ab.txt 2>&1
done
