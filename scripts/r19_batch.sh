python -m pytest tests/test_gpu_ls.py tests/test_gpu_engine.py tests/test_gpu_engine_large.py tests/test_gpu_heavy.py -q -x > gpurun_out/r19_tests.log 2>&1; tail -3 gpurun_out/r19_tests.log
python scripts/bench_core.py --out gpurun_out/r19_bench_core.jsonl > /dev/null 2>&1
python -c "
import json
for l in open('gpurun_out/r19_bench_core.jsonl'):
    d=json.loads(l)
    if d['case'] in ('one_flip_pass','one_two_swap','mis_trajectory'): print(d['case'], d['n'], round(d['ref_cpu_us'],1), round(d['gpu_1_us'],1), round(d['speedup_1'],2), round(d['speedup_b'],1))"
for v in 0 11; do python scripts/smallb_probe.py --graph c4 --chains 16,128 --traj 0 --variant $v; done
for v in 0 12; do python scripts/smallb_probe.py --graph c3 --chains 256 --traj 0 --variant $v; python scripts/smallb_probe.py --graph c5 --chains 16,64 --traj 0 --variant $v; done
python scripts/ls_bench.py
python scripts/e2e_breakdown.py 4
