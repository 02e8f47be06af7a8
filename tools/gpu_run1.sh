set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -30
timeout 600 python tools/select_methods.py --dims 3 --points 1e7 --out gpurun_out/select_r1a.jsonl 2>&1 | tail -70
