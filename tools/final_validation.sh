# Single-B200 evidence run for profiles/r02 (gpurun): GPU tests, smoke, bench lines, launch list, step ncu capture.
python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/final_bench_bf16.json 2> gpurun_out/final_bench_bf16.err
python bench.py --precision mixed > gpurun_out/final_bench_mixed.json 2> gpurun_out/final_bench_mixed.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --no-extras --no-factored --steps 2 --warmup 1 > gpurun_out/final_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -o /tmp/final_step python tools/profile_step.py > gpurun_out/final_ncu_step.log 2>&1
ncu -i /tmp/final_step.ncu-rep --page raw --csv > gpurun_out/final_step_raw.csv 2>/dev/null
ncu --set full --clock-control none --import-source on -k regex:graph_csr_kernel -c 1 -o gpurun_out/final_graph python tools/profile_step.py > gpurun_out/final_ncu_graph.log 2>&1
ls -la gpurun_out; tail -1 gpurun_out/final_pytest_gpu.log
