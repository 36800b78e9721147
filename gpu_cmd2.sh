mkdir -p gpurun_out/s24
timeout 1500 python -m pytest tests -m gpu -x -q -k "detector or frcnn or cfg4 or bench_config or cfg5" > gpurun_out/s24/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/s24/pytest_gpu.log
for r in 1 2; do
python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/s24/bench_cfg4.json 2> gpurun_out/s24/bench.err
python -c "import json;d=json.load(open('gpurun_out/s24/bench_cfg4.json'));print('base',d['value'],d['ms_per_step'],{k:round(v['ms'],3) for k,v in d['roofline']['by_kind'].items()})"
done
CFG=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s24/launches_cfg4.csv python tools/run_step.py 1 > /dev/null 2>&1
