#!/bin/bash
# variant choice vs problem size (tools/size_probe.py, tuning build)
mkdir -p gpurun_out/size
HEXFUSE_B200_LIB=$PWD/paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so timeout 1500 python tools/size_probe.py > gpurun_out/size/size_probe.jsonl 2> gpurun_out/size/err; echo rc=$?; tail -3 gpurun_out/size/err
