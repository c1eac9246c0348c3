mkdir -p gpurun_out
python -c "from paper_2603_05800_b200 import build; build.build(); from oracle import oracle; oracle.build()" > gpurun_out/r3l_build.log 2>&1
SW_DEBUG=1 SW_TRACE=1 timeout 300 python tools/one_step.py C3 2 > gpurun_out/r3l_c3_debug.txt 2>&1
timeout 600 python bench.py --config C3 > gpurun_out/r3l_bench_c3.json 2> gpurun_out/r3l_bench_c3.err
timeout 600 python bench.py > gpurun_out/r3l_bench.json 2> gpurun_out/r3l_bench.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3l_pytest.log
timeout 300 python tools/stream_bench.py C2 > gpurun_out/r3l_stream.txt 2>&1; timeout 300 python tools/stream_bench.py C3 >> gpurun_out/r3l_stream.txt 2>&1
echo done
