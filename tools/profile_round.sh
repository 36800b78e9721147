#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench lines of every config, the
# reference arm, the ncu launch list of one cfg4 step, per-config GEMM DRAM traffic,
# per-layer-class GEMM attribution tables, and ncu --set full captures of cfg4's
# largest GEMM launch, the fused stem kernels and RoIAlign.  Outputs under
# gpurun_out/<tag>/ (copy summaries to profiles/).
# usage: bash tools/profile_round.sh r2
tag=${1:-r2}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
python bench.py > $out/bench_cfg4.json 2> $out/bench.err
for c in 2 3 5; do python bench.py --no-cpu --cfg $c > $out/bench_cfg$c.json 2>> $out/bench.err; done
python bench.py --impl reference --steps 4 --warmup 1 > $out/bench_reference.json 2>> $out/bench.err
CFG=4 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg4.csv \
    python tools/run_step.py 1 > /dev/null 2>&1
for c in 4 2 3 5; do
  CFG=$c ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:gemel_gemm --csv --log-file $out/traffic_cfg$c.csv python tools/run_step.py 1 > /dev/null 2>&1
  rm -rf $out/trace$c
  CFG=$c python tools/trace_step.py $out/trace$c > /dev/null 2>> $out/trace.err
  python tools/gemm_attribution.py $out/trace$c > $out/gemm_classes_cfg$c.json 2>> $out/trace.err
  rm -f $out/trace$c/*.bin
done
CFG=4 ncu --set full --import-source on --clock-control none -k regex:gemel_gemm_sm100 -s 1 -c 1 \
    -o $out/ncu_cfg4_gemm python tools/run_step.py 1 > $out/ncu_full.log 2>&1
ncu -i $out/ncu_cfg4_gemm.ncu-rep --page raw --csv > $out/ncu_cfg4_gemm_raw.csv 2>/dev/null
rm -f $out/ncu_cfg4_gemm.ncu-rep
for k in stem_kernel roi_align rpn_nms topk_kernel; do
  CFG=4 ncu --set full --clock-control none -k regex:$k -c 2 -o $out/ncu_$k python tools/run_step.py 1 > /dev/null 2>&1
  ncu -i $out/ncu_$k.ncu-rep --page raw --csv > $out/ncu_${k}_raw.csv 2>/dev/null
  rm -f $out/ncu_$k.ncu-rep
done
