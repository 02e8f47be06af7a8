#!/bin/bash
# full lines-variant sweep of the tuning build (variants 0-27, padded x-rows included)
mkdir -p gpurun_out/sel3
HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so timeout 2400 python tools/select_methods.py --dims 3,2 --no-planar --no-unfused --points 1e7 --out gpurun_out/sel3/sel.jsonl > /dev/null 2>gpurun_out/sel3/sel.err
echo "sel rc=$?"; tail -3 gpurun_out/sel3/sel.err
HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "lines_variants" > gpurun_out/sel3/pytest_tuning.log 2>&1; tail -1 gpurun_out/sel3/pytest_tuning.log
