#!/bin/bash
# time tools/profile_render.py with every variants/*/libvoxvid_b200.so (and the default build)
echo "== default"; python tools/profile_render.py --frames 10 "$@"
for d in variants/*/; do echo "== $d"; VV_LIB_PATH=$d/libvoxvid_b200.so python tools/profile_render.py --frames 10 "$@"; done
