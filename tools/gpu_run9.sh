timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 1500 python tools/select_methods.py --dims 3,2 --points 1e7 --no-unfused --out gpurun_out/select_r1f.jsonl > /dev/null 2>&1
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/select_r1f.jsonl')]
best={}
for r in rows:
    k=(r['d'],r['p'],r['precision'])
    if r['method']=='planar': continue
    print(k, r['variant'], r['kernel'], round(r['alg_GBps']), round(r['spread'],2))
PY
