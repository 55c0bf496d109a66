#!/bin/bash
# usage: tools/libswap.sh <variant .so> <command...>  (tuning experiments only)
cp paper_2112_00132_b200/libatos.so /tmp/libatos_main.so
cp "$1" paper_2112_00132_b200/libatos.so
shift
"$@"
cp /tmp/libatos_main.so paper_2112_00132_b200/libatos.so
