#!/bin/bash
# Round-2 measurement set on one B200 (production build): GPU suite, smoke, every BASELINE workload,
# the reference arm, the ncu launch list of the default bench (per-launch time + DRAM bytes), one ncu
# --set full capture of the dominant kernel.
set -o pipefail
O=gpurun_out/${OUT:-bench_r02}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
for w in config1 config3 config4 config5; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?"
done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file $O/ncu_launches_config2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_bench.json 2>&1
echo "ncu list rc=$?"
python tools/ncu_traffic.py $O/ncu_launches_config2.csv $O/bench_config2.json $O/ncu_traffic.json 3 > $O/ncu_traffic.txt 2>&1; echo "traffic rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hf_lines -s 1 -c 1 -o $O/full_dom \
  python tools/prof_one.py --d 3 --p 6 --prec fp64 --variant -1 --launches 2 > $O/full_dom.log 2>&1
python tools/ncu_brief.py $O/full_dom.ncu-rep > $O/full_dom_brief.txt 2>&1
ncu -i $O/full_dom.ncu-rep --page raw --csv > $O/full_dom_raw.csv 2>/dev/null
rm -f $O/full_dom.ncu-rep
echo done
