#!/bin/bash
O=gpurun_out/r02j; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
timeout 600 python bench.py --workload config3 --no-cpu > $O/bench_config3.json 2> $O/bench_config3.err; echo "bench3 rc=$?"
timeout 900 python tools/bench_fr.py --out $O/bench_fr.jsonl > /dev/null 2> $O/bench_fr.err; echo "fr rc=$?"
