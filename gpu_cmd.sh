timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 300 python tools/trace_step.py gpurun_out/trace 2>&1 | tail -1 | python -c "import json,sys; print([(l['kind'], round(l['ms']*1000,1)) for l in json.loads(sys.stdin.read())])"
