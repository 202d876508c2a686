#!/bin/bash
# Build git revision $1 (default HEAD) of libbolt.so into paper_1706_10283_b200/libbolt_base.so
# (same-box A/B timing against the working tree: BOLT_LIB=libbolt_base.so).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/bolt_base_wt
rm -rf "$WT"; git -C "$ROOT" worktree prune
git -C "$ROOT" worktree add -f --detach "$WT" "$REV" >/dev/null
(cd "$WT" && python -m paper_1706_10283_b200.build >/dev/null)
cp "$WT/paper_1706_10283_b200/libbolt.so" "$ROOT/paper_1706_10283_b200/libbolt_base.so"
git -C "$ROOT" worktree remove --force "$WT"
echo "$ROOT/paper_1706_10283_b200/libbolt_base.so <- $(git -C "$ROOT" rev-parse --short "$REV")"
