#!/bin/bash
# Round 2: component-split variants (19-23) on the tuning build: parity (incl. bit identity with
# the one-thread-per-line variants) and a timing sweep against variants 0/1/2/7/3.
O=gpurun_out/r02i; mkdir -p $O
TL=paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so
HEXFUSE_B200_LIB=$TL timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "lines_variants or component_split or pipe_many" > $O/pytest_cs.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_cs.log
HEXFUSE_B200_LIB=$TL timeout 1500 python tools/select_methods.py --points 1e7 --no-unfused --no-planar --variants 0,1,2,3,7,19,20,21,22,23 --out $O/select_cs.jsonl > /dev/null 2> $O/select_cs.err; echo "select rc=$?"
