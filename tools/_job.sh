GSS_LIB=$PWD/build_old/libgss.so timeout 600 python -m pytest tests/test_gpu_ring_protocol.py -x -q -m gpu 2>&1 | tail -2
