#!/bin/bash
# Run tools/probe.py against the in-tree library and each build/*/libotfgpu.so variant.
for v in "" build/*/; do
  if [ -z "$v" ]; then echo "== in-tree"; unset OTFGPU_LIB_OVERRIDE; else echo "== $v"; export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; fi
  timeout 300 python tools/probe.py "$@" 2>&1 | tail -4
done
