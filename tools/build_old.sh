#!/bin/bash
# Build the library from git HEAD into _lib/libintattn_b200_old.so (A/B baseline; development tool).
set -e
d=$(mktemp -d)
git archive HEAD paper_2511_21513_b200/csrc include | tar -x -C $d
make -s -C $d/paper_2511_21513_b200/csrc OUT=$PWD/paper_2511_21513_b200/_lib/libintattn_b200_old.so $PWD/paper_2511_21513_b200/_lib/libintattn_b200_old.so
rm -rf $d
