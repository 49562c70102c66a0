#!/bin/bash
# time the cfg2 step with every libwsb variant in tools/variants/
cd "$(dirname "$0")/.."
for so in tools/variants/*.so; do
  echo -n "$(basename $so): "
  WSB_LIB=$PWD/$so timeout 120 python tools/profile_step.py --steps 4 "$@" 2>&1 | tail -1
done
