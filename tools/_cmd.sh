timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/step_timing.py > gpurun_out/st.log 2>&1
