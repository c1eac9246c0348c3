# C3 big scan pass (pass 3 of the first step) under ncu --set full, with source
mkdir -p gpurun_out
python -c "from paper_2603_05800_b200 import build; build.build(); from oracle import oracle; oracle.build()" > gpurun_out/r3h_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/r3h_c3_scan3 python tools/one_step.py C3 1 > gpurun_out/r3h_ncu_scan.log 2>&1
echo done
