# 4-GPU evidence run for profiles/r02 (gpurun --gpus 4): torchrun bench at N=2/4 and the NCCL multi-rank tests.
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/final_bench_n2.json 2> gpurun_out/final_bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 > gpurun_out/final_bench_n4.json 2> gpurun_out/final_bench_n4.err
python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/final_pytest_mr4.log 2>&1
tail -1 gpurun_out/final_pytest_mr4.log; tail -c 300 gpurun_out/final_bench_n4.json
