#!/bin/bash
# Decode A/B on one box: the in-tree build (variants $VARIANTS) against the
# prebuilt _variants/*.so (run under gpurun from the repo root).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
args=""
for v in ${VARIANTS:-0}; do args="$args paper_2510_10302_b200/libspmoe.so:$v"; done
for f in _variants/*.so; do args="$args $f"; done
timeout 600 python tools/decode_ab.py $args
