#!/bin/bash
# Round 2: selection re-measured on the tuning build (CUDA events + ncu counters incl. the planar
# kernels' bank conflicts); small-problem probe (fixed cost per launch, occupancy cap).
O=gpurun_out/r02g; mkdir -p $O
TL=paper_2107_14027_b200/lib_tuning/libhexfuse_b200.so
HEXFUSE_B200_LIB=$TL timeout 1800 python tools/select_methods.py --points 1e7 --no-unfused --out $O/select.jsonl > /dev/null 2> $O/select.err; echo "select rc=$?"
HEXFUSE_B200_LIB=$TL timeout 1500 ncu --metrics $(python tools/select_ncu.py --metrics) --clock-control none --csv \
   --log-file $O/sel_ncu.csv python tools/select_ncu.py --launch $O/sel_launches.json > $O/sel_ncu.log 2>&1; echo "ncu rc=$?"
python tools/select_ncu.py --parse $O/sel_ncu.csv $O/sel_launches.json > $O/sel_ncu.jsonl 2> $O/sel_ncu_parse.err; echo "parse rc=$?"
timeout 600 python tools/small_probe.py > $O/small_probe.jsonl 2> $O/small_probe.err; echo "probe rc=$?"
for c in 3 4 6 8; do
  PROBE_TAG=maxcta$c HF_LINES_MAXCTA=$c HEXFUSE_B200_LIB=paper_2107_14027_b200/lib_alt/libhexfuse_b200.so timeout 600 python tools/small_probe.py >> $O/small_probe_cap.jsonl 2>> $O/small_probe_cap.err
done
echo done
