# shard processes on one B200 under a private MPS daemon (multi-process C5
# path: CUDA IPC, system-scope flags); grids capped so the kernels co-reside
mkdir -p gpurun_out /tmp/mps_pipe /tmp/mps_log
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
nvidia-cuda-mps-control -d && echo mps_started
for w in 2 4; do
  g=$((148 / w))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 \
    --master-port $((29700 + w)) tools/c5_multiproc.py --same-gpu --grid $g --sim 12000000 --p 64 \
    > gpurun_out/c5_mps_$w.log 2>&1; echo world=$w rc=$?
  grep -E '^\{' gpurun_out/c5_mps_$w.log
done
echo quit | nvidia-cuda-mps-control; echo mps_stopped
