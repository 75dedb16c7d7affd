#!/bin/bash
# rebuild libpdg.so locally (the snapshot ships it), then run a command on the GPU box
set -e
make -s -C "$(dirname "$0")/../paper_2007_04881_b200/csrc" -j8 > /dev/null
exec /usr/local/graft/bin/gpurun "$@"
