#!/bin/bash
# Build the committed HEAD (or a given revision) of the library into build/base/
# for A/B runs against the working tree:  tools/build_base.sh [rev]
set -e
rev=${1:-HEAD}
root=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/vfmm_base && mkdir -p /tmp/vfmm_base
git -C "$root" archive "$rev" paper_0809_1810_b200/csrc include | tar -x -C /tmp/vfmm_base
mkdir -p "$root/build/base"
make -C /tmp/vfmm_base/paper_0809_1810_b200/csrc -j8 OUT="$root/build/base/libvfmm.so" > /dev/null
echo "$root/build/base/libvfmm.so"
