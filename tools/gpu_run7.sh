timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lines or pipe or config1" 2>&1 | tail -3
timeout 900 python tools/select_methods.py --dims 3 --points 1e7 --no-unfused --out gpurun_out/select_r1d.jsonl 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    if r['method']=='planar': continue
    print(r['d'],r['p'],r['precision'],r['variant'],r['kernel'],round(r['alg_GBps']),r['regs'])
"
