#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench lines, reference arm,
# per-config lines, swap comparison, ncu launch list + one full capture of the
# dominant GEMM launch, summarised into profiles/<tag>_*.
# usage: bash tools/profile_round.sh r1
tag=${1:-r1}
out=gpurun_out/$tag
mkdir -p $out
python bench.py > $out/bench.json 2> $out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference.json 2>> $out/bench.err
for c in 3 4 5; do python bench.py --no-cpu --cfg $c > $out/bench_cfg$c.json 2>> $out/bench.err; done
for m in none cross; do
  python bench.py --no-cpu --cfg 3 --merge $m --budget-frac 0.5 --steps 10 > $out/bench_cfg3_budget50_$m.json 2>> $out/bench.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemel_gemm -s 1 -c 1 -o $out/prof_gemm \
    python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/summarize_profiles.py $out $tag > /dev/null
tail -c 400 $out/bench.json
