mkdir -p gpurun_out/s12
GEMEL_STEM=1 timeout 900 python -m pytest tests -m gpu -x -q -k "cfg1 or mixed or cfg2_small or bench_config or detector_teacher" > gpurun_out/s12/pytest_gpu_stem1.log 2>&1
tail -n 2 gpurun_out/s12/pytest_gpu_stem1.log
GEMEL_STEM=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/s12/bench_cfg4_stem1.json 2> gpurun_out/s12/bench.err
python -c "import json;d=json.load(open('gpurun_out/s12/bench_cfg4_stem1.json'));print(d['value'],d['ms_per_step'],{k:round(v['ms'],3) for k,v in d['roofline']['by_kind'].items()})"
CFG=4 GEMEL_STEM=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:stem_kernel -c 2 -o gpurun_out/s12/stem python tools/run_step.py 1 > gpurun_out/s12/ncu2.log 2>&1
ncu -i gpurun_out/s12/stem.ncu-rep --page raw --csv > gpurun_out/s12/stem_raw.csv 2>/dev/null
ncu -i gpurun_out/s12/stem.ncu-rep --page source --csv > gpurun_out/s12/stem_source.csv 2>/dev/null
rm -f gpurun_out/s12/stem.ncu-rep
rm -rf gpurun_out/s12/trace4; CFG=4 timeout 300 python tools/trace_step.py gpurun_out/s12/trace4 > /dev/null 2> gpurun_out/s12/trace.err
for l in 1 3 5; do python tools/trace_report.py gpurun_out/s12/trace4 $l 200 > gpurun_out/s12/trace_l$l.txt 2>> gpurun_out/s12/trace.err; done
python tools/gemm_attribution.py gpurun_out/s12/trace4 > gpurun_out/s12/gemm_classes_cfg4.json 2>> gpurun_out/s12/trace.err
rm -f gpurun_out/s12/trace4/*.bin
