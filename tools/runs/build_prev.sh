#!/bin/bash
# Build libpcb200.so from a commit (default HEAD) into ablib/prev for same-box A/B runs.
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2311_04934_b200/csrc include | tar -x -C "$TMP"
make -C "$TMP/paper_2311_04934_b200/csrc" -j8 > "$TMP/build.log" 2>&1 || { tail -20 "$TMP/build.log"; exit 1; }
mkdir -p "$ROOT/ablib/prev"
cp "$TMP/paper_2311_04934_b200/lib/libpcb200.so" "$ROOT/ablib/prev/libpcb200.so"
rm -rf "$TMP"
echo "ablib/prev <- $(git -C "$ROOT" rev-parse --short "$REV")"
