#!/bin/bash
# full GPU suite, then the planar methods against lines variant 0 (production build)
mkdir -p gpurun_out/planar
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/planar/pytest.log 2>&1; tail -2 gpurun_out/planar/pytest.log
timeout 900 python tools/select_methods.py --dims 3 --variants 0 --no-unfused --points 1e7 --out gpurun_out/planar/sel.jsonl > /dev/null 2>gpurun_out/planar/sel.err
echo "sel rc=$?"; tail -3 gpurun_out/planar/sel.err
