#!/bin/bash
O=gpurun_out/r02h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dependent_back_to_back" > $O/pytest_pdl.log 2>&1; echo "pdl test rc=$?"; tail -1 $O/pytest_pdl.log
timeout 600 python bench.py > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
timeout 300 python bench.py --workload config1 --no-cpu > $O/bench_config1.json 2> $O/bench_config1.err; echo "c1 rc=$?"
bash tools/gpu_sanitize_r02.sh
