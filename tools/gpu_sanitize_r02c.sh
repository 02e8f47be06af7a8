#!/bin/bash
# compute-sanitizer over this session's new paths: padded grouped chunks and vectorised
# element-major x-lines (groups 1, 2), the tile ring (variant 24), the mapped kernel's
# last-sweep epilogue, the reworked planar kernels.
O=gpurun_out/san_r02c; mkdir -p $O
CS=compute-sanitizer
KG='lines_groups_fp64_p3 or lines_groups_fp32_p4'
timeout 2400 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mapped.py -q -x -k "tile_ring or $KG or planar or mapped_curved" > $O/memcheck.log 2>&1; echo "mem rc=$?"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "tile_ring and not fp32" > $O/racecheck_ring.log 2>&1; echo "race ring rc=$?"
timeout 2400 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mapped.py -q -x -k "$KG or planar_random or boxes" > $O/racecheck.log 2>&1; echo "race rc=$?"
timeout 2400 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_mapped.py -q -x -k "tile_ring or $KG or boxes" > $O/synccheck.log 2>&1; echo "sync rc=$?"
timeout 1200 $CS --tool initcheck python -m pytest tests/test_gpu_parity.py -q -x -k "$KG" > $O/initcheck.log 2>&1; echo "init rc=$?"
for f in $O/*.log; do echo "$f: $(grep -E 'SUMMARY|passed|failed' $f | tr '\n' ' ')"; done
