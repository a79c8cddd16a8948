#!/bin/bash
# build the working tree's libsgad.so with extra nvcc flags into variants/<name>.so
#   tools/build_flags.sh name -DSGAD_OS_MINB=3 ...
set -e
name=$1; shift
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I include "$@" -o variants/$name.so paper_2603_21055_b200/csrc/*.cu
