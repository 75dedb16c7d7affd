#!/bin/bash
# A/B the element kernel of two source trees on the same box:
#   tools/ab.sh <git-rev>   (builds <rev> into ab_base/ here, ships it with the snapshot)
# then on the box:  bash tools/ab_run.sh
set -e
REV=${1:-HEAD}
rm -rf ab_base && mkdir ab_base
git archive "$REV" | tar -x -C ab_base
make -s -C ab_base/paper_2007_04881_b200/csrc -j8 > /dev/null
echo "built $REV into ab_base/"
