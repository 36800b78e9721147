mkdir -p gpurun_out/s17
python __graft_entry__.py smoke > gpurun_out/s17/smoke.log 2>&1; tail -n 1 gpurun_out/s17/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s17/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/s17/pytest_gpu.log
python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/s17/bench_cfg4.json 2> gpurun_out/s17/bench.err
python -c "import json;d=json.load(open('gpurun_out/s17/bench_cfg4.json'));print('base',d['value'],d['ms_per_step'],d['e2e'],{k:round(v['ms'],3) for k,v in d['roofline']['by_kind'].items()})"
