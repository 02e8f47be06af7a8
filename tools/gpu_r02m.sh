#!/bin/bash
# Round 2: the reworked guarded path (per-element bases + cp.async word copies) on groups no
# other path takes (odd strides), a misaligned base, and config 2 (production paths unchanged).
O=gpurun_out/r02m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "caller_groups or misaligned or groups_fp64 or tile_mode" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 900 python tools/group_sweep.py --d 3 --groups 3,5,15 > $O/groups_odd_d3.jsonl 2> $O/groups_odd.err; echo "sweep rc=$?"
timeout 600 python tools/group_sweep.py --d 2 --groups 3,7,15 > $O/groups_odd_d2.jsonl 2>> $O/groups_odd.err; echo "sweep2 rc=$?"
timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_config2.json 2> $O/bench_config2.err; echo "bench rc=$?"
