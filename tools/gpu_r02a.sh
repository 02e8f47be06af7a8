#!/bin/bash
# Round 2: scale parity tests, the new bench contract (parity field, reference arm without the B200 library).
set -o pipefail
O=gpurun_out/r02a; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x > $O/pytest_scale.log 2>&1; tail -3 $O/pytest_scale.log
timeout 600 python bench.py > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
timeout 900 python bench.py --workload config5 > $O/bench_config5.json 2> $O/bench_config5.err; echo "bench5 rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
grep -c libhexfuse /proc/self/maps >/dev/null
