python profiles/gs_small.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gs_launches.csv python profiles/gs_small.py > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/gs_launches.csv | head -30
