timeout 120 ./build/gemm_selftest | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -2
for ms in 1 8; do GEMEL_MAX_SPLIT=$ms timeout 300 python tools/trace_step.py gpurun_out/trace$ms 2>&1 | tail -1 | python -c "import json,sys; print('split $ms', [(l['kind'], round(l['ms']*1000,1)) for l in json.loads(sys.stdin.read())])"; done
for ms in 1 8; do GEMEL_MAX_SPLIT=$ms timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench split $ms', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"; done
