#!/bin/bash
# Per-kernel registers / spills / shared memory of libbolt.so (demangled, filtered by regex $1)
cuobjdump --dump-resource-usage "$(dirname "$0")/../paper_1706_10283_b200/libbolt.so" 2>/dev/null | \
  grep -E "Function|REG" | paste - - | sed -E 's/\s+/ /g' | \
  sed -E 's/Function ([^:]*):.*REG:([0-9]+) STACK:([0-9]+) SHARED:([0-9]+) LOCAL:([0-9]+).*/\1 REG=\2 STACK=\3 SHARED=\4 LOCAL=\5/' | \
  while read f rest; do echo "$(echo $f | c++filt | sed -E 's/bolt::\(anonymous namespace\):://; s/\(.*//' | cut -c1-70) $rest"; done | grep -E "${1:-.}"
