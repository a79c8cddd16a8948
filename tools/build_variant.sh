#!/bin/bash
# build libsgad.so from a git revision into variants/<name>.so (A/B timing)
set -e
rev=$1; name=$2
tmp=$(mktemp -d)
git -C /root/repo worktree add -q --detach "$tmp" "$rev"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I "$tmp/include" -o /root/repo/variants/$name.so "$tmp"/paper_2603_21055_b200/csrc/*.cu
git -C /root/repo worktree remove --force "$tmp"
