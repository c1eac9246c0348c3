mkdir -p gpurun_out
python -c "from paper_2603_05800_b200 import build; build.build(); from oracle import oracle; oracle.build()" > gpurun_out/r3d_build.log 2>&1
SW_DEBUG=1 SW_TRACE=1 timeout 300 python tools/one_step.py C3 2 > gpurun_out/r3d_c3_debug.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3d_c3_launches.csv python tools/one_step.py C3 1 > gpurun_out/r3d_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/r3d_c3_scan python tools/one_step.py C3 2 > gpurun_out/r3d_ncu_scan.log 2>&1
echo done
