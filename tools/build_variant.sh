#!/bin/bash
# Build the working-tree library with extra -D flags into _lib/<name>.so (development tool).
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
name=$1; shift
make -s -C paper_2511_21513_b200/csrc OUT=../_lib/$name.so ../_lib/$name.so NVFLAGS_EXTRA="$*"
