timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 1500 python tools/select_methods.py --dims 3,2 --points 1e7 --no-unfused --out gpurun_out/select_r1g.jsonl > /dev/null 2>&1
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/select_r1g.jsonl')]
best={}
for r in rows:
    k=(r['d'],r['p'],r['precision'])
    if r['method']=='planar': continue
    if k not in best or r['alg_GBps']>best[k]['alg_GBps']: best[k]=r
    print(k, r['variant'], r['kernel'], round(r['alg_GBps']))
print("BEST")
for k in sorted(best): print(k, best[k]['variant'], best[k]['kernel'], round(best[k]['alg_GBps']))
PY
