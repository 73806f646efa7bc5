# A/B timing of libvdmc variants in one gpurun call:
#   bash tools/ab.sh TAG default VARIANT...   (variants: paper_2201_11655_b200/lib/libvdmc_VARIANT.so,
#   built by tools/build_variant.sh).  AB_CONFIGS="cfg4 cfg5" selects the workloads; AB_PARITY=1 also
#   runs a GPU parity subset against each variant.
O=gpurun_out/$1; shift; mkdir -p $O
for v in "$@"; do
  if [ $v = default ]; then unset VDMC_LIB; else export VDMC_LIB=$PWD/paper_2201_11655_b200/lib/libvdmc_$v.so; fi
  echo "== $v" >> $O/ab.txt
  for c in ${AB_CONFIGS:-cfg4}; do timeout 600 python tools/phase_probe.py $c 4 quick >> $O/ab.txt 2>&1; done
  if [ "${AB_PARITY:-0}" = 1 ]; then
    timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_undirected.py -x -q -k "small_fixtures or heavy_and_light or scaled" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
  fi
done
