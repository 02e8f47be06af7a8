# full GPU test suite + the default bench line (tools/README.md)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -c 3000 gpurun_out/bench_full.json
