#!/bin/bash
# selection refresh with the padded variants: timing sweep + ncu counters of every candidate
# (d3 and d2, tuning build, one box), then the tuning build's variant parity
O=gpurun_out/sel4; mkdir -p $O
export HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so
timeout 2400 python tools/select_methods.py --dims 3,2 --no-planar --no-unfused --points 1e7 --out $O/sel.jsonl > /dev/null 2>$O/sel.err; echo "sel rc=$?"
timeout 3000 ncu --metrics $(python tools/select_ncu.py --metrics) --clock-control none --csv --log-file $O/sel_ncu.csv \
  python tools/select_ncu.py --launch $O/sel_launches.json --dims 3,2 > $O/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/select_ncu.py --parse $O/sel_ncu.csv $O/sel_launches.json > $O/sel_ncu.jsonl 2> $O/parse.err; echo "parse rc=$?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "lines_variants" > $O/pytest_tuning.log 2>&1; tail -1 $O/pytest_tuning.log
