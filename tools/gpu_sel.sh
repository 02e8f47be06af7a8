#!/bin/bash
# GPU parity suite, then the full lines-variant sweep of the current build.
mkdir -p gpurun_out/sel
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/sel/pytest.log 2>&1; tail -2 gpurun_out/sel/pytest.log
timeout 1800 python tools/select_methods.py --dims 3,2 --no-planar --no-unfused --points 1e7 --out gpurun_out/sel/sel.jsonl > /dev/null 2>gpurun_out/sel/sel.err
echo "sel rc=$?"
