#!/bin/bash
# A/B only.  Make a variant copy of csrc/ and build it as a separate library:
#   bash tools/variant.sh new NAME     -> build/variants/NAME/csrc (edit it)
#   bash tools/variant.sh build NAME   -> build/variants/libNAME.so
set -e
cd "$(dirname "$0")/.."
V=build/variants
mkdir -p $V/include
cp include/*.h $V/include/
case $1 in
  new) rm -rf $V/$2; mkdir -p $V/$2; cp -r paper_2503_01199_b200/csrc $V/$2/csrc ;;
  build) make -s -C $V/$2/csrc OUT=../../lib$2.so OBJDIR=../obj HDRS="common.cuh onesweep.cuh" && echo built $V/lib$2.so ;;
esac
