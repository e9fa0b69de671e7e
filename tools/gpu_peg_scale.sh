#!/bin/bash
export MBP_PEG_DEBUG=2
timeout 600 python tools/peg_gpu_time.py 65536 32768 1 2>&1 | tail -2
timeout 1200 python tools/peg_gpu_time.py 262144 131072 1 2>&1 | tail -2
