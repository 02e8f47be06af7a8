#!/bin/bash
# planar parity, then the lines-variant + planar sweep of the tuning build (selection refresh
# after the vectorised element-major x-lines changed the NE = 1 variants)
mkdir -p gpurun_out/sel2
timeout 900 python -m pytest tests -q -m gpu -x -k "planar" > gpurun_out/sel2/pytest_planar.log 2>&1; tail -2 gpurun_out/sel2/pytest_planar.log
HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so timeout 2400 python tools/select_methods.py --dims 3,2 --no-unfused --points 1e7 --out gpurun_out/sel2/sel.jsonl > /dev/null 2>gpurun_out/sel2/sel.err
echo "sel rc=$?"; tail -3 gpurun_out/sel2/sel.err
