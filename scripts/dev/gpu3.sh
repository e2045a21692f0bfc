mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "linear" > gpurun_out/pytest_linear.log 2>&1; tail -3 gpurun_out/pytest_linear.log
timeout 600 python scripts/dev/gemv_sweep.py ${1:-1,8,16,32} > gpurun_out/sweep.log 2>&1; grep -v relerr gpurun_out/sweep.log | grep '"pdl": true'; grep relerr gpurun_out/sweep.log | sort -t: -k5 | tail -2
if [ -n "$2" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 40 -c 1 -o gpurun_out/prof_$2 python scripts/ncu_target.py $3 $4 $5 > gpurun_out/ncu_$2.log 2>&1; tail -2 gpurun_out/ncu_$2.log
fi
