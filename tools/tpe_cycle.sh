#!/bin/bash
# GPU cycle for the thread-per-element variant: parity, sweep (fused vs tpe), C2 bench, ncu of k_tpe
TAG=${1:-x}
python -m pytest tests -m gpu -q -x -k "variant or tpe or loopback" 2>&1 | tail -2
python bench.py --sweep --sweep-variants 1 3 > gpurun_out/sweep_$TAG.jsonl 2>&1; head -8 gpurun_out/sweep_$TAG.jsonl | cut -c1-120
python bench.py --no-cpu --no-solve --no-e2e --variant 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cut -c1-200 gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
if [ "${2:-ncu}" = "ncu" ]; then
for N in 3 4; do
ncu --set full --clock-control none --import-source on -k regex:k_tpe -s 1 -c 2 -o gpurun_out/prof_${TAG}_N$N python tools/prof_run.py --N $N --variant 3 --pcg 2 > gpurun_out/ncu_${TAG}_N$N.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_N$N.log
done
fi
