#!/bin/bash
# A/B library variants (tools only): tools/variants.sh NAME "-DFLAG=V ..." builds
# paper_2603_10242_b200/lib/libacegpu.so with EXTRA flags into variants/NAME/
# (then restores the default build). Run probes with ACEGPU_LIB=variants/NAME/libacegpu.so.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
P=$ROOT/paper_2603_10242_b200
name=$1; shift
rm -f $P/build/*.o
make -C $P -j16 EXTRA="$*" > /tmp/variant_$name.log 2>&1 || { tail -20 /tmp/variant_$name.log; exit 1; }
mkdir -p $ROOT/variants/$name && cp $P/lib/libacegpu.so $ROOT/variants/$name/
rm -f $P/build/*.o
make -C $P -j16 > /dev/null 2>&1
mkdir -p $ROOT/variants/base && cp $P/lib/libacegpu.so $ROOT/variants/base/
echo "built variants/$name"
