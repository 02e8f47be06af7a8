#!/bin/bash
# final measurement set of the round: GPU suite, smoke, every workload, reference arm, ncu launch
# list + full capture (tools/gpu_bench_r02.sh), then the extension sweeps (FR, mapped; burst protocol)
OUT=${OUT:-bench_final} bash tools/gpu_bench_r02.sh
O=gpurun_out/${OUT:-bench_final}
timeout 900 python tools/bench_fr.py --dims 3,2 --out $O/ext_fr.jsonl > /dev/null 2> $O/ext_fr.err; echo "fr rc=$?"
timeout 900 python tools/bench_mapped.py --out $O/ext_mapped.jsonl > /dev/null 2> $O/ext_mapped.err; echo "mapped rc=$?"
