nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py > gpurun_out/bench_s2.json 2> gpurun_out/bench_s2.err; cut -c1-400 gpurun_out/bench_s2.json; tail -2 gpurun_out/bench_s2.err
python bench.py --sweep > gpurun_out/sweep_s2.jsonl 2>&1; cut -c1-160 gpurun_out/sweep_s2.jsonl
