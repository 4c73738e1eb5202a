# round-2 final measurements (inside gpurun, repo root)
set -x
python -m pytest tests -m gpu -q > gpurun_out/gputest_v21.log 2>&1; tail -2 gpurun_out/gputest_v21.log
python bench.py > gpurun_out/bench_config2_v21.json 2> gpurun_out/bench_config2_v21.err
python bench.py --impl reference > gpurun_out/bench_reference_v21.json 2> gpurun_out/bench_reference_v21.err
python bench.py --config 3 > gpurun_out/bench_config3_v21.json 2> gpurun_out/bench_config3_v21.err
python bench.py --config 4 --steps 3 > gpurun_out/bench_config4_v21.json 2> gpurun_out/bench_config4_v21.err
bash tools/dram_bench.sh 2 2048
bash tools/ncu_k1.sh 2 64 k1_config2_v21
bash tools/ncu_k1.sh 3 128 k1_config3_v21
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_seeds64_v21.csv python bench.py --steps 2 --warmup 1 --seeds 64 --no-cpu-baseline > gpurun_out/launches.log 2>&1
tail -c 300 gpurun_out/bench_config2_v21.json; tail -c 300 gpurun_out/bench_config3_v21.json
