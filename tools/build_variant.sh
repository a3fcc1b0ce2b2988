#!/bin/bash
# Build libspmoe.so of git ref $1 into _variants/$2.so (A/B timing on one box:
# tools/decode_ab.py loads several builds side by side).
set -e
ref=$1; name=$2
tmp=$(mktemp -d)
git archive "$ref" | tar -x -C "$tmp"
(cd "$tmp" && python -c "from paper_2510_10302_b200.build import build; build(force=True)")
mkdir -p _variants
cp "$tmp/paper_2510_10302_b200/libspmoe.so" "_variants/$name.so"
rm -rf "$tmp"
echo "_variants/$name.so"
