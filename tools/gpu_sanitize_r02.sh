#!/bin/bash
# Round 2: compute-sanitizer over the kernels added this round -- the staged FR correction with
# ghost layers (ADVICE), tile mode (TMA tensor copies) and grouped chunks, the staged unfused
# stage 3, the blob path (host).  racecheck + synccheck + memcheck on small parity cases.
O=gpurun_out/san_r02; mkdir -p $O
CS=compute-sanitizer
K_FR='test_fr_layer_partitions_with_ghosts and (2-True or 5-True or 8-True)'
K_TILE='test_caller_groups_d2 or test_tile_mode_with_misaligned'
K_UNF='test_nonunit_jac_fp64'
timeout 1200 $CS --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_fr.py -q -x -k "$K_FR" > $O/racecheck_fr_staged.log 2>&1; echo "race fr rc=$?"
timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_fr.py -q -x -k "$K_FR" > $O/synccheck_fr_staged.log 2>&1; echo "sync fr rc=$?"
timeout 1200 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "$K_TILE" > $O/racecheck_tile_grouped.log 2>&1; echo "race tile rc=$?"
timeout 1200 $CS --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "$K_TILE" > $O/synccheck_tile_grouped.log 2>&1; echo "sync tile rc=$?"
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "$K_TILE or $K_UNF" > $O/memcheck_tile_unfused.log 2>&1; echo "mem rc=$?"
timeout 1200 $CS --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "$K_UNF" > $O/racecheck_unfused.log 2>&1; echo "race unf rc=$?"
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_host.py -q -x -k "blob or in_place" > $O/memcheck_host_blob.log 2>&1; echo "mem host rc=$?"
for f in $O/*.log; do echo "$f: $(grep -E 'SUMMARY|passed|failed' $f | tr '\n' ' ')"; done
