mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemel_gemm -s 5 -c 1 -o gpurun_out/prof_mega python tools/run_step.py 3 > gpurun_out/ncu_mega.log 2>&1; tail -2 gpurun_out/ncu_mega.log
