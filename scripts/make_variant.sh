#!/bin/bash
# Snapshot the built package into variants/<name>/ (timing A/B of two builds on one box):
#   scripts/make_variant.sh NAME            (current working tree build)
# then on the GPU:  python scripts/ab_variants.py NAME1 NAME2 ...
set -e
cd "$(dirname "$0")/.."
rm -rf "variants/$1"
mkdir -p "variants/$1"
cp -r paper_2604_13327_b200 "variants/$1/"
rm -rf "variants/$1/paper_2604_13327_b200/csrc"
