set -x
python tools/gnn_ab.py 14 > gpurun_out/ab6.log 2>&1
python bench.py --no-extras > gpurun_out/b15.log 2>gpurun_out/b15.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 3 --warmup 3 --no-extras --no-factored --screen-compounds 4916 > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none -k regex:"graph_csr|conv_umma|dense_tf32|gnn_mma|voxelize|dense_kernel|topk|best" -c 12 -o /tmp/step_bf16 python tools/profile_step.py > gpurun_out/ncu_step.log 2>&1
ncu -i /tmp/step_bf16.ncu-rep --page raw --csv > gpurun_out/step_bf16_raw.csv 2>>gpurun_out/ncu_step.log
FS_PROFILE_PRECISION=mixed ncu --set full --clock-control none -k regex:gnn_mma_kernel -c 1 -o /tmp/gnn_mixed python tools/profile_step.py >> gpurun_out/ncu_step.log 2>&1
ncu -i /tmp/gnn_mixed.ncu-rep --page raw --csv > gpurun_out/gnn_mixed_raw.csv 2>>gpurun_out/ncu_step.log
ls -la gpurun_out
