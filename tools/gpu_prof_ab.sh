for lib in abtest/lib_head.so paper_2107_14027_b200/lib/libhexfuse_b200.so; do
tag=$(basename $lib .so)
HEXFUSE_B200_LIB=$PWD/$lib timeout 300 ncu --set full --import-source on --clock-control none -k regex:hf_lines -s 1 -c 1 -o gpurun_out/ab_$tag python tools/prof_one.py --d 3 --p 3 --prec fp64 --variant 0 --launches 2 > /dev/null 2>&1
done
ls gpurun_out
