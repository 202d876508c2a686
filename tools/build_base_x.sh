#!/bin/bash
# Build git revision $1 (default HEAD) as libbolt_base.so and its diagnostic
# (BOLT_XMODE) twin libbolt_x_base.so, for same-box A/B runs.
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/bolt_base_wt
rm -rf "$WT"; git -C "$ROOT" worktree prune
git -C "$ROOT" worktree add -f --detach "$WT" "$REV" >/dev/null
(cd "$WT" && python -m paper_1706_10283_b200.build >/dev/null && python -m paper_1706_10283_b200.build --xmode >/dev/null && python -m paper_1706_10283_b200.build --profile >/dev/null)
cp "$WT/paper_1706_10283_b200/libbolt.so" "$ROOT/paper_1706_10283_b200/libbolt_base.so"
cp "$WT/paper_1706_10283_b200/libbolt_x.so" "$ROOT/paper_1706_10283_b200/libbolt_x_base.so"
cp "$WT/paper_1706_10283_b200/libbolt_prof.so" "$ROOT/paper_1706_10283_b200/libbolt_prof_base.so"
git -C "$ROOT" worktree remove --force "$WT"
echo "libbolt_base.so + libbolt_x_base.so <- $(git -C "$ROOT" rev-parse --short "$REV")"
