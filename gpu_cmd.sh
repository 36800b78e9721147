timeout 120 ./build/gemm_selftest | tail -1
timeout 60 ./build/gemm_selftest bench | grep grouped
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -2
timeout 300 python tools/trace_step.py gpurun_out/trace 2>&1 | tail -1 | python -c "import json,sys; print([(l['kind'], round(l['ms']*1000,1)) for l in json.loads(sys.stdin.read())])"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
