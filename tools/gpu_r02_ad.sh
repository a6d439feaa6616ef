timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02ad_launches_c3.csv python tools/step_probe.py c3 > /dev/null 2>&1; echo rc=$?
