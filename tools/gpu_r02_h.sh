#!/bin/bash
# strategy sweep (config line + fixed chi = 100), oracle baselines on the GPU box host
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --configs c2,c3,c4,c5,c5_256 --strategies sequential --steps 5 > gpurun_out/r02h_sweep_seq.jsonl 2> gpurun_out/r02h_sweep.err
timeout 1500 python tools/sweep.py --configs c2,c3,c4,c5 --strategies reduced --steps 3 > gpurun_out/r02h_sweep_red.jsonl 2>> gpurun_out/r02h_sweep.err
timeout 1500 python tools/sweep.py --configs c2,c3,c4 --strategies standard --steps 2 > gpurun_out/r02h_sweep_std.jsonl 2>> gpurun_out/r02h_sweep.err
timeout 1500 python tools/sweep.py --configs D4_chi100,D6_chi100,D8_chi100,D10_chi100 --strategies sequential,reduced --steps 3 > gpurun_out/r02h_sweep_chi100.jsonl 2>> gpurun_out/r02h_sweep.err
timeout 900 python tools/sweep.py --configs D4_chi100,D6_chi100,D8_chi100 --strategies standard --steps 2 >> gpurun_out/r02h_sweep_chi100.jsonl 2>> gpurun_out/r02h_sweep.err
timeout 1800 python tools/oracle_baselines.py --configs c2,c3,c4,c5 > gpurun_out/r02h_oracle_baselines.jsonl 2> gpurun_out/r02h_oracle.err
