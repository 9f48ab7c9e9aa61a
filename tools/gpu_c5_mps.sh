# two shard processes on one B200 under MPS (multi-process C5 path: CUDA IPC,
# system-scope flags); each rank's grid capped at 74 CTAs so both co-reside
mkdir -p gpurun_out /tmp/mps_pipe /tmp/mps_log
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
nvidia-cuda-mps-control -d && echo mps_started
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29531 tools/c5_multiproc.py --same-gpu --grid 74 > gpurun_out/c5_multiproc.log 2>&1
echo rc=$?
grep -E '^\{' gpurun_out/c5_multiproc.log; tail -5 gpurun_out/c5_multiproc.log | grep -v '^{'
echo quit | nvidia-cuda-mps-control; echo mps_stopped
