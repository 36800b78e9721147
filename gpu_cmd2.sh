mkdir -p gpurun_out/s8
python -m pytest tests -m gpu -x -q -k "detector or frcnn or cfg4 or mixed or cfg5" > gpurun_out/s8/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/s8/pytest_gpu.log
python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/s8/bench_cfg4.json 2> gpurun_out/s8/bench.err
CFG=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s8/launches_cfg4.csv python tools/run_step.py 1 > gpurun_out/s8/ncu1.log 2>&1
CFG=4 GEMEL_STEM=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:stem_kernel -c 2 -o gpurun_out/s8/stem python tools/run_step.py 1 > gpurun_out/s8/ncu2.log 2>&1
ncu -i gpurun_out/s8/stem.ncu-rep --page raw --csv > gpurun_out/s8/stem_raw.csv 2>/dev/null
ncu -i gpurun_out/s8/stem.ncu-rep --page source --csv > gpurun_out/s8/stem_source.csv 2>/dev/null
rm -f gpurun_out/s8/stem.ncu-rep
for i in 17 18; do timeout 120 ncu --set full --clock-control none -k regex:gemel_gemm -c 1 -o gpurun_out/s8/micro$i build/gemm_selftest bench $i > gpurun_out/s8/micro$i.log 2>&1; ncu -i gpurun_out/s8/micro$i.ncu-rep --page raw --csv > gpurun_out/s8/micro${i}_raw.csv 2>/dev/null; rm -f gpurun_out/s8/micro$i.ncu-rep; done
