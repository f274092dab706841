#!/bin/bash
# two ranks sharing the one GPU (gloo on CUDA tensors): the sharded code paths on the device
export PYTHONDONTWRITEBYTECODE=1
SBT_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config hooi --no-cpu --steps 2 > gpurun_out/mr_hooi.json 2> gpurun_out/mr_hooi.err; tail -c 600 gpurun_out/mr_hooi.json; tail -5 gpurun_out/mr_hooi.err
SBT_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config small --no-e2e --no-cpu --steps 3 > gpurun_out/mr_small.json 2> gpurun_out/mr_small.err; tail -c 300 gpurun_out/mr_small.json; tail -3 gpurun_out/mr_small.err
