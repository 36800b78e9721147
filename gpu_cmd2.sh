#!/bin/bash
mkdir -p gpurun_out/r2prof
ST=build/gemm_selftest
for i in 0 1 2 3 4 5 6 7 8; do echo "== micro $i"; timeout 60 $ST bench $i 2>&1 | grep -E "grouped|case|tiles"; done > gpurun_out/r2prof/micro.txt 2>&1
for c in 4 2 3 5; do
  rm -rf gpurun_out/r2prof/trace$c
  CFG=$c timeout 300 python tools/trace_step.py gpurun_out/r2prof/trace$c > /dev/null 2> gpurun_out/r2prof/trace$c.err
  python tools/gemm_attribution.py gpurun_out/r2prof/trace$c > gpurun_out/r2prof/attr_cfg$c.json 2>> gpurun_out/r2prof/trace$c.err
  rm -f gpurun_out/r2prof/trace$c/*.bin
done
