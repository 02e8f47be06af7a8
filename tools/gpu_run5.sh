set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv
free -g | head -2
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -8
timeout 120 python tools/pcie_probe.py
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r1b_config2.json 2> gpurun_out/bench_r1b_config2.err
timeout 300 python bench.py --workload config1 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_r1b_config1.json 2>&1
timeout 300 python bench.py --workload config3 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_r1b_config3.json 2>&1
timeout 300 python bench.py --workload config4 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_r1b_config4.json 2>&1
timeout 600 python bench.py --workload config5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r1b_config5.json 2>&1
timeout 300 python bench.py --impl reference --steps 50 --warmup 5 > gpurun_out/bench_r1b_reference.json 2>&1
for f in gpurun_out/bench_r1b_*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ['value','ms_per_step','impl']}, d.get('roofline',{}).get('frac'), d.get('roofline',{}).get('step_aggregate_frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d.get('unfused'), d.get('clocks'))
"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench_r1b.log 2>&1
tail -2 gpurun_out/ncu_launch_bench_r1b.log
