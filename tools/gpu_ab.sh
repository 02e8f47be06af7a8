for lib in abtest/lib_head.so paper_2107_14027_b200/lib/libhexfuse_b200.so abtest/lib_head.so paper_2107_14027_b200/lib/libhexfuse_b200.so; do
echo "== $lib"
HEXFUSE_B200_LIB=$PWD/$lib timeout 600 python tools/select_methods.py --dims 3 --ps 1,3,4,5,6 --variants 0,1,3,5 --no-planar --no-unfused --points 1e7 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(r['p'],r['precision'],r['variant'],round(r['alg_GBps']),r['regs'],r['smem'])
"
done
