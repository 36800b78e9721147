mkdir -p gpurun_out/s22
timeout 120 build/gemm_selftest > gpurun_out/s22/selftest.log 2>&1; tail -n 1 gpurun_out/s22/selftest.log
CG=2 timeout 120 build/gemm_selftest > gpurun_out/s22/selftest_cg2.log 2>&1; tail -n 1 gpurun_out/s22/selftest_cg2.log
{
for i in 16 17 18 19 11 15 3 12; do echo "== micro $i"; timeout 60 build/gemm_selftest bench $i 2>&1 | grep -E "grouped"; done
for dbg in 64 67; do echo "== micro 16 dbg $dbg"; timeout 60 build/gemm_selftest bench 16 $dbg 2>&1 | grep -E "grouped"; done
} > gpurun_out/s22/micro.txt 2>&1
cat gpurun_out/s22/micro.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s22/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/s22/pytest_gpu.log
for r in 1 2; do
python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/s22/bench_cfg4.json 2> gpurun_out/s22/bench.err
python -c "import json;d=json.load(open('gpurun_out/s22/bench_cfg4.json'));print('base',d['value'],d['ms_per_step'],{k:round(v['ms'],3) for k,v in d['roofline']['by_kind'].items()})"
done
