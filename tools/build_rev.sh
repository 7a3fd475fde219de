#!/bin/bash
# Build libqtt.so of a git revision into tools/libqtt_<name>.so for same-box A/B timing:
#   tools/build_rev.sh <rev> <name>;  then QTT_LIB=$PWD/tools/libqtt_<name>.so python ...
set -e
cd "$(dirname "$0")/.."
rev=$1; name=$2
wt=/tmp/qtt_wt_$name
rm -rf "$wt"
git worktree add -f --detach "$wt" "$rev" >/dev/null 2>&1
make -C "$wt/paper_2501_12151_b200/csrc" -j8 >/dev/null
cp "$wt/paper_2501_12151_b200/libqtt.so" "tools/libqtt_$name.so"
git worktree remove --force "$wt"
echo "tools/libqtt_$name.so"
