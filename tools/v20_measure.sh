# round-2 final measurements (inside gpurun, repo root)
set -x
python bench.py > gpurun_out/bench_config2_v20.json 2> gpurun_out/bench_config2_v20.err
python bench.py --config 3 > gpurun_out/bench_config3_v20.json 2> gpurun_out/bench_config3_v20.err
python bench.py --config 4 --steps 3 > gpurun_out/bench_config4_v20.json 2> gpurun_out/bench_config4_v20.err
bash tools/dram_bench.sh 3 4096
bash tools/ncu_k1.sh 3 128 k1_config3_v20
tail -c 300 gpurun_out/bench_config2_v20.json; tail -c 300 gpurun_out/bench_config3_v20.json
