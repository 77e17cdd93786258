python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err; tail -3 gpurun_out/b1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --strong cfg4 --no-cpu > gpurun_out/b2.json 2> gpurun_out/b2.err; tail -3 gpurun_out/b2.err
