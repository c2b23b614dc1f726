#!/bin/bash
# Build libmgb200.so of a git revision into ab/<name>.so (same-box A/B timing via
# MGB_LIB_OVERRIDE). Usage: tools/ab_build.sh REV NAME
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/mgb_wt_$name
rm -rf "$wt"; git -C "$root" worktree prune
git -C "$root" worktree add -f --detach "$wt" "$rev" >/dev/null
make -C "$wt/paper_2408_03204_b200/csrc" -j8 >/dev/null
mkdir -p "$root/ab"
cp "$wt/paper_2408_03204_b200/libmgb200.so" "$root/ab/$name.so"
git -C "$root" worktree remove --force "$wt"
echo "built ab/$name.so from $(git -C "$root" rev-parse --short "$rev")"
