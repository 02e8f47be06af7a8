set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "group or misaligned or guarded or tile" 2>&1 | tail -5
timeout 600 python tools/group_sweep.py --d 3 --groups 1,2,4,8 > gpurun_out/gs_pad_d3.jsonl 2> gpurun_out/gs_pad_d3.err
timeout 600 python tools/group_sweep.py --d 2 --groups 1,2,4,8 > gpurun_out/gs_pad_d2.jsonl 2> gpurun_out/gs_pad_d2.err
tail -3 gpurun_out/gs_pad_d3.err
