#!/bin/bash
# Extensions: GPU parity of the mapped-element and FR-stage kernels and their timing sweeps.
O=gpurun_out/ext2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fr.py tests/test_gpu_mapped.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 900 python tools/bench_fr.py --out $O/bench_fr.jsonl > /dev/null 2> $O/bench_fr.err; echo "fr rc=$?"
timeout 900 python tools/bench_mapped.py --dims 3 --out $O/bench_mapped.jsonl > /dev/null 2> $O/bench_mapped.err; echo "mapped rc=$?"
