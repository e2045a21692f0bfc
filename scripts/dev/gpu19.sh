timeout 300 python -m pytest tests -x -q -m gpu -k "chain or linear_vs_oracle or partition" > gpurun_out/p.log 2>&1; tail -3 gpurun_out/p.log
timeout 600 python bench.py --steps 20 --warmup 5 --sweep "1,2,4,8,16" --cpu-seconds 1 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -c 1200 gpurun_out/bench3.json
