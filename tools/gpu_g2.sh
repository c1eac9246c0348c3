# ncu captures of the hot kernels, exported on the box (raw metrics + source page as CSV)
set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/store_pattern tools/microbench/store_pattern.cu && /tmp/store_pattern > gpurun_out/g2_store_pattern.txt 2>&1
cap() {  # name, kernel regex, skip, cmd...
  local n=$1 k=$2 s=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$n "$@" > gpurun_out/${n}_ncu.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > gpurun_out/${n}_raw.csv 2>&1
  ncu -i /tmp/$n.ncu-rep --page source --csv --print-source sass > gpurun_out/${n}_sass.csv 2>&1
  ncu -i /tmp/$n.ncu-rep --page details > gpurun_out/${n}_details.txt 2>&1
}
cap g2_eval_c2 eval_kernel 2 python tools/one_step.py C2 3
cap g2_eval_c5 eval_kernel 2 python tools/one_step_c5.py
cap g2_scan_c3 scan_kernel 8 python tools/one_step.py C3 3
SW_DEBUG=1 timeout 300 python tools/one_step.py C3 2 > gpurun_out/g2_c3_debug.txt 2>&1
ls -la gpurun_out; du -sh gpurun_out
echo done
