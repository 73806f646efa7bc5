#!/bin/bash
# A/B of prebuilt variant libs only (no build, no tests): bash tools/run_ab.sh TAG VARIANT...
O=gpurun_out/$1; shift; mkdir -p $O
AB_CONFIGS="${AB_CONFIGS:-cfg4 cfg5}" bash tools/ab.sh ${O#gpurun_out/} "$@"
