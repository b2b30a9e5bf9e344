timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_f1.json 2> gpurun_out/bench_f1.err; cut -c1-300 gpurun_out/bench_f1.json; tail -3 gpurun_out/bench_f1.err
timeout 600 python bench.py --config C4 --steps 300 --no-cpu --no-solve > gpurun_out/bench_f1_C4.json 2> gpurun_out/bench_f1_C4.err; tail -2 gpurun_out/bench_f1_C4.err
for v in 2 4; do timeout 600 python bench.py --config C4 --steps 300 --no-cpu --no-solve --no-e2e --variant $v > gpurun_out/bench_f1_C4_v$v.json 2>&1; done
python -c "
import json
for t in ('f1','f1_C4','f1_C4_v2','f1_C4_v4'):
    d=json.load(open('gpurun_out/bench_%s.json'%t)); print(t, d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['ax_only'])
"
