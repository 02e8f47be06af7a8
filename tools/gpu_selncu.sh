#!/bin/bash
# ncu counters of every d3 selection candidate on the current tuning build (tools/select_ncu.py)
O=gpurun_out/selncu; mkdir -p $O
export HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so
timeout 3000 ncu --metrics $(python tools/select_ncu.py --metrics) --clock-control none --csv --log-file $O/sel_ncu.csv \
  python tools/select_ncu.py --launch $O/sel_launches.json --dims 3 > $O/launch.log 2>&1; echo "ncu rc=$?"
python tools/select_ncu.py --parse $O/sel_ncu.csv $O/sel_launches.json > $O/sel_ncu_d3.jsonl 2> $O/parse.err; echo "parse rc=$?"
