set -x
for cfg in "3 6 fp32 3" "3 6 fp32 0" "3 6 fp64 3" "3 4 fp32 3"; do set -- $cfg
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hf_lines -s 1 -c 1 -o gpurun_out/prof_d$1p$2$3v$4 python tools/prof_one.py --d $1 --p $2 --prec $3 --variant $4 --launches 2 > /dev/null 2>&1
done
timeout 900 python tools/select_methods.py --dims 2 --points 2e7 --no-unfused --out gpurun_out/select_r1_d2.jsonl 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r['d'],r['p'],r['precision'],r['method'],r['variant'],r['kernel'],round(r['alg_GBps']),r['regs'],r['block'],r['smem'])
"
ls gpurun_out
