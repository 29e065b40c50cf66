#!/bin/bash
# build libfovnet (and the oracle) here, then run the given command on a B200 via gpurun
set -e
cd /root/repo
make -s -C paper_2209_09965_b200/csrc -j8 > /tmp/build.log 2>&1 || { grep -i error -A3 /tmp/build.log | head -30; exit 1; }
make -s -C oracle > /dev/null
exec /usr/local/graft/bin/gpurun --timeout "${GPU_TIMEOUT:-2400}" -- "$@"
