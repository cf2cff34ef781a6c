timeout 700 python -m pytest tests -q -m gpu --timeout 400 -x > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_run.py grover20 60 > gpurun_out/ncu_all.csv 2>&1
