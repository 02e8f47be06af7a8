#!/bin/bash
# padded x-row chunks (lines variants 25-27): parity, then timing + bank conflicts against the
# unpadded chunks of the same size at d3 p3
O=gpurun_out/xpad; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "lines_variants" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 900 python tools/select_methods.py --dims 3 --ps 3 --variants 7,25,1,26,0,27 --no-planar --no-unfused --points 1e7 --out $O/sel.jsonl > /dev/null 2> $O/sel.err; echo "sel rc=$?"
timeout 900 ncu --metrics $(python tools/select_ncu.py --metrics) --clock-control none --csv --log-file $O/ncu.csv \
  python tools/select_ncu.py --launch $O/launches.json --dims 3 --variants 7,25,1,26,0,27 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/select_ncu.py --parse $O/ncu.csv $O/launches.json > $O/ncu.jsonl 2> $O/parse.err
