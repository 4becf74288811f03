#!/bin/bash
# Full round evidence: smoke, GPU tests, bench per config, launch list + ncu full capture of cfg3/cfg5 level passes.
set -u
mkdir -p gpurun_out
bash tools/gpu_check.sh
CFG=3 SKIP=3 TAG=cfg3 bash tools/ncu_level.sh
CFG=5 SKIP=5 TAG=cfg5 bash tools/ncu_level.sh
CFG=2 SKIP=0 TAG=cfg2 bash tools/ncu_level.sh
