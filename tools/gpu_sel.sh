#!/bin/bash
# GPU parity suite on the production build + smoke, then the full lines-variant
# sweep of the tuning build (make tuning).
mkdir -p gpurun_out/sel
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/sel/pytest.log 2>&1; tail -2 gpurun_out/sel/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sel/smoke.log 2>&1; echo "smoke rc=$?"
HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so timeout 1800 python tools/select_methods.py --dims 3,2 --no-planar --no-unfused --points 1e7 --out gpurun_out/sel/sel.jsonl > /dev/null 2>gpurun_out/sel/sel.err
echo "sel rc=$?"
