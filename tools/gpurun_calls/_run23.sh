python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r23_build.log 2>&1
RESOCT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/peer_overhead.py > gpurun_out/r23_peer.log 2>&1; echo rc=$?; grep '^{' gpurun_out/r23_peer.log; tail -3 gpurun_out/r23_peer.log
