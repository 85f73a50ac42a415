#!/bin/bash
# build in this container, then run a script on the GPU box (one call)
set -e
cd /root/repo
python paper_2504_08624_b200/_build.py > /dev/null
/usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-900} -- "bash $1" 2>&1 | tail -${TAIL:-40}
