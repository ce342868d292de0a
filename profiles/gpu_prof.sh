mkdir -p gpurun_out
# launch list: both kernels of a K2V2 and a K3V4 config-2 layer
timeout 300 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/tc_launches.csv python profiles/drive_attend.py > gpurun_out/drive.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_tc -s 1 -c 1 -o gpurun_out/tc_prof python profiles/drive_attend.py 0 > gpurun_out/drive2.log 2>&1
timeout 300 python profiles/attend_time.py > gpurun_out/attend_time.log 2>&1
KVMIX_TC=0 timeout 300 python profiles/attend_time.py > gpurun_out/attend_time_notc.log 2>&1
