#!/bin/bash
# cross-compile tuning builds of liboec into tune/ (tile parameters as -D)
set -e
cd "$(dirname "$0")/.."
b() { python -m paper_2005_13014_b200.build --out=tune/$1.so "${@:2}" > /dev/null; echo "$1 ${@:2}"; }
b h_2_8_3_6  -DHD_V=2 -DHD_JB=8 -DHD_S=3 -DHD_NW=6 &
b h_2_4_4_6  -DHD_V=2 -DHD_JB=4 -DHD_S=4 -DHD_NW=6 &
b h_2_16_2_5 -DHD_V=2 -DHD_JB=16 -DHD_S=2 -DHD_NW=5 &
b h_4_8_2_5  -DHD_V=4 -DHD_JB=8 -DHD_S=2 -DHD_NW=5 &
wait
b h_1_8_4_8  -DHD_V=1 -DHD_JB=8 -DHD_S=4 -DHD_NW=8 &
b h_2_8_2_8  -DHD_V=2 -DHD_JB=8 -DHD_S=2 -DHD_NW=8 &
b v_64_2_4   -DVA_NC=64 -DVA_LB=2 -DVA_S=4 &
b v_32_8_2   -DVA_NC=32 -DVA_LB=8 -DVA_S=2 &
wait
b v_64_8_2   -DVA_NC=64 -DVA_LB=8 -DVA_S=2 &
b v_128_4_2  -DVA_NC=128 -DVA_LB=4 -DVA_S=2 &
b v_32_4_4   -DVA_NC=32 -DVA_LB=4 -DVA_S=4 &
b v_64_4_3   -DVA_NC=64 -DVA_LB=4 -DVA_S=3 &
wait
