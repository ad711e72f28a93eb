GSN=12830211 GSM=64 python profiles/gs_small.py
GSN=12830211 GSM=64 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/gs_launches64.csv python profiles/gs_small.py > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/gs_launches64.csv | head -30
