set -x
python bench.py > gpurun_out/bench_config2_v19.json 2> gpurun_out/bench_config2_v19.err
python bench.py --impl reference > gpurun_out/bench_reference_v19.json 2> gpurun_out/bench_reference_v19.err
python bench.py --config 3 > gpurun_out/bench_config3_v19.json 2> gpurun_out/bench_config3_v19.err
python bench.py --config 4 --steps 3 > gpurun_out/bench_config4_v19.json 2> gpurun_out/bench_config4_v19.err
bash tools/dram_bench.sh 2 2048
bash tools/dram_bench.sh 2 2048 --records
bash tools/dram_bench.sh 3 4096
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_seeds64_v19.csv python bench.py --steps 2 --warmup 1 --seeds 64 --no-cpu-baseline > gpurun_out/launches.log 2>&1
bash tools/ncu_k1.sh 3 32 k1_config3_v19
tail -c 300 gpurun_out/bench_config2_v19.json; tail -c 200 gpurun_out/bench_config3_v19.json
