#!/bin/bash
# padded chunks with k-plane padding for one-element chunks (d3 p4-p7): parity of the
# tuning build's padded variants, timing + ncu against the unpadded ones
O=gpurun_out/xpad2; mkdir -p $O
export HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "lines_variants" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 900 python tools/select_methods.py --dims 3 --ps 4,5,6,7 --variants 7,25,1,26,0,27,15,3 --no-planar --no-unfused --points 1e7 --out $O/sel.jsonl > /dev/null 2> $O/sel.err; echo "sel rc=$?"
timeout 900 ncu --metrics $(python tools/select_ncu.py --metrics) --clock-control none --csv --log-file $O/ncu.csv \
  python tools/select_ncu.py --launch $O/launches.json --dims 3 --variants 7,25,1,26,0,27 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/select_ncu.py --parse $O/ncu.csv $O/launches.json > $O/ncu.jsonl 2> $O/parse.err
