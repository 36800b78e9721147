mkdir -p gpurun_out/r1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/ -q -m gpu 2>&1 | tail -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/r1/bench.json 2> gpurun_out/r1/bench.err; cat gpurun_out/r1/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1/bench_ref.json 2>&1; tail -1 gpurun_out/r1/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1/launches.csv python tools/run_step.py 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemel_gemm -s 5 -c 1 -o gpurun_out/r1/prof_mega python tools/run_step.py 3 > gpurun_out/r1/ncu_mega.log 2>&1
tail -1 gpurun_out/r1/ncu_mega.log
