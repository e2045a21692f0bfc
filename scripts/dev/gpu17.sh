timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv python scripts/dev/dec_prof.py > /dev/null 2>&1; echo rc=$?
