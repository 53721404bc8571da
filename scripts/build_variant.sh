#!/bin/bash
# Build libseakv.so with extra nvcc flags into scripts/ab/libseakv_<name>.so (A/B runs:
# SKV_LIB_PATH=scripts/ab/libseakv_<name>.so python ...).  Usage: build_variant.sh <name> <flags>
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$TMP/pkg" "$TMP/include"
cp -r "$ROOT/paper_2504_15720_b200/csrc" "$TMP/pkg/csrc"
cp -r "$ROOT/include/." "$TMP/include/"
rm -rf "$TMP/pkg/csrc/build"
# the Makefile reads ../../include and writes ../libseakv.so relative to csrc
make -s -C "$TMP/pkg/csrc" SKV_EXTRA="$*" > /dev/null
mkdir -p "$ROOT/scripts/ab"
cp "$TMP/pkg/libseakv.so" "$ROOT/scripts/ab/libseakv_$NAME.so"
rm -rf "$TMP"
echo "built scripts/ab/libseakv_$NAME.so ($*)"
