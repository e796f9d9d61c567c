#!/bin/bash
# Build the backend at a git revision (or the working tree: "WT") into ab/lib<name>.so
# usage: tools/build_variant.sh <rev|WT> <name>
set -e
cd "$(dirname "$0")/.."
rev=$1; name=$2; tmp=$(mktemp -d)
if [ "$rev" = "WT" ]; then
  mkdir -p "$tmp/paper_2601_03159_b200"; cp -r paper_2601_03159_b200/csrc "$tmp/paper_2601_03159_b200/"; cp -r include "$tmp/"
else
  git archive "$rev" paper_2601_03159_b200/csrc include | tar -x -C "$tmp"
fi
mkdir -p ab
make -s -C "$tmp/paper_2601_03159_b200/csrc" OUT="$PWD/ab/lib$name.so" > /dev/null
rm -rf "$tmp"; ls -la ab/lib$name.so
