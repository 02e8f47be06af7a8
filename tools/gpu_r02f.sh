#!/bin/bash
# Round 2: programmatic dependent launch A/B (HF_PDL=0/1) on configs 1, 2, 3; unfused grid-stride flux; GPU suite.
O=gpurun_out/r02f; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for w in config1 config2 config3; do
  for i in 1 2; do
    HF_PDL=0 timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-parity > $O/${w}_pdl0_$i.json 2>$O/${w}_pdl0_$i.err
    HF_PDL=1 timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-parity > $O/${w}_pdl1_$i.json 2>$O/${w}_pdl1_$i.err
  done
done
echo ab done
timeout 300 python bench.py --workload config4 --no-cpu --no-e2e > $O/bench_config4.json 2> $O/bench_config4.err; echo "c4 rc=$?"
