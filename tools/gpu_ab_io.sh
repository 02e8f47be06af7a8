#!/bin/bash
# Parity of the current build, then lines-variant sweeps for: the base library,
# the current library and the IO-only build (chunk traffic without the sweeps).
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/ab/pytest.log 2>&1; tail -2 gpurun_out/ab/pytest.log
for tag in base:abtest/lib_base.so new:paper_2107_14027_b200/lib/libhexfuse_b200.so io:abtest/io/libhexfuse_b200.so; do
  name=${tag%%:*}; lib=${tag#*:}
  HEXFUSE_B200_LIB=$PWD/$lib timeout 1200 python tools/select_methods.py --dims 3,2 --no-planar --no-unfused --points 1e7 --out gpurun_out/ab/sel_$name.jsonl > /dev/null 2>&1
  echo "$name rc=$?"
done
