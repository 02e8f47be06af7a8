#!/bin/bash
# FR right-hand side A/B on one box: current library vs lib_alt, d3 sweep (tools/bench_fr.py),
# then the FR parity suite on the current library
O=gpurun_out/fr_ab; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fr.py tests/test_gpu_peer.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for v in new alt new2 alt2; do
  case $v in new*) L=lib;; alt*) L=lib_alt;; esac
  HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/$L/libhexfuse_b200.so timeout 900 python tools/bench_fr.py --dims 3 --out $O/$v.jsonl > /dev/null 2> $O/$v.err; echo "$v rc=$?"
done
