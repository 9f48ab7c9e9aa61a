# the bench's multi-rank path (C2 replicas, C4 tasks over ranks, C5 shards with
# the in-kernel exchange) with 2 ranks sharing one B200 under a private MPS
# daemon; grids capped so the two ranks' kernels co-reside
mkdir -p gpurun_out /tmp/mps_pipe2 /tmp/mps_log2
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe2 CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log2
nvidia-cuda-mps-control -d && echo mps_started
GSS_MAX_GRID=74 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 --steps 2 --warmup 3 \
  --c2-n 2000000 --c2-p 500 --c3-p 0 --no-c1 --c4-n 200000 --c4-p 200 --c5-rows 2000000 --c5-p 64 \
  --no-cpu-baseline --no-parity > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo rc=$?
tail -3 gpurun_out/bench_2rank.err
cat gpurun_out/bench_2rank.json
echo quit | nvidia-cuda-mps-control; echo mps_stopped
