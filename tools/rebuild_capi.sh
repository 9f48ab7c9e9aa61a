#!/bin/bash
# incremental rebuild of libgss.so after editing gss_capi.cu only (the full build is __graft_entry__.build())
set -e
R=/root/repo; O=$R/build/obj
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 177 -c $R/paper_2204_08183_b200/csrc/gss_capi.cu -o $O/gss_capi.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared $O/gss_aux.o $O/gss_capi.o $O/gss_comm.o $O/gss_cycle.o $O/gss_ingest.o $O/gss_separated.o $O/gss_simgen.o -o $R/paper_2204_08183_b200/libgss.so
