#!/bin/bash
# compute-sanitizer memcheck over the GPU suites of the final library (parity, FR, mapped, host path,
# drop-in, blob), and racecheck over the parity suite's lines kernels
O=gpurun_out/san_final; mkdir -p $O
CS=compute-sanitizer
timeout 5400 $CS --tool memcheck --leak-check no python -m pytest tests/test_gpu_parity.py tests/test_gpu_fr.py \
  tests/test_gpu_mapped.py tests/test_gpu_host.py tests/test_gpu_dropin.py -q -m gpu > $O/memcheck.log 2>&1; echo "mem rc=$?"
timeout 3600 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -m gpu -k "lines_d3 or lines_d2 or padded or tile_ring or caller_groups_d2" > $O/racecheck.log 2>&1; echo "race rc=$?"
for f in $O/*.log; do echo "$f: $(grep -E 'SUMMARY|passed|failed' $f | tr '\n' ' ')"; done
