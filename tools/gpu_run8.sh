timeout 1200 python tools/select_methods.py --dims 3,2 --points 1e7 --no-unfused --out gpurun_out/select_r1e.jsonl 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r['d'],r['p'],r['precision'],r['method'][:3],r['variant'],r['kernel'],round(r['alg_GBps']),round(r['spread'],2),r['regs'])
"
