#!/bin/bash
O=gpurun_out/r02k; mkdir -p $O
timeout 300 python tools/pcie_probe.py > $O/pcie.txt 2>&1; echo "pcie rc=$?"; tail -3 $O/pcie.txt
timeout 600 python bench.py --no-cpu --no-parity > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
TL=paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so
HEXFUSE_B200_LIB=$TL timeout 900 python tools/tile_probe.py --d 3 --ps 4,5,6 --groups 8,16,24,32,64 --variants 7,1,0,2,22,20,19,21 > $O/tile_probe_cs.jsonl 2> $O/tile_probe_cs.err; echo "probe rc=$?"
