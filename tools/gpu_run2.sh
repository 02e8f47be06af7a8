set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r1_config2.json 2> gpurun_out/bench_r1_config2.err
tail -c 3000 gpurun_out/bench_r1_config2.json
timeout 300 python bench.py --workload config4 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_r1_config4.json 2>&1
tail -c 1500 gpurun_out/bench_r1_config4.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r1_reference.json 2>&1
cat gpurun_out/bench_r1_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1
tail -3 gpurun_out/ncu_launch_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hf_lines_kernel -s 36 -c 12 -o gpurun_out/prof_r1_lines python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" > gpurun_out/host_cpu.txt
ls -la gpurun_out
