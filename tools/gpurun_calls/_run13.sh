python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r13_build.log 2>&1
export RESOCT_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --exchange peer --no-e2e > gpurun_out/r13_peer.log 2>&1; echo "peer rc=$?"
tail -c 1500 gpurun_out/r13_peer.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 4 --warmup 3 --exchange nccl --no-e2e > gpurun_out/r13_nccl.log 2>&1; echo "nccl-path rc=$?"
tail -c 1500 gpurun_out/r13_nccl.log
timeout 600 python -m pytest tests/test_gpu_peer.py -q -x > gpurun_out/r13_peertest.log 2>&1; tail -3 gpurun_out/r13_peertest.log
