PFFMG_VC_SEQ=1 python tools/prof_vcycle.py cfg2 > gpurun_out/vcseq_cfg2.txt 2>&1
PFFMG_VC_SEQ=1 python tools/prof_vcycle.py cfg3 > gpurun_out/vcseq_cfg3.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --strong cfg4 --no-cpu > gpurun_out/b2.json 2> gpurun_out/b2.err; echo "rc=$?" >> gpurun_out/b2.err
