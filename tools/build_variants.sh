#!/bin/bash
# cross-compile tuning builds of liboec into tune/ (tile parameters as -D)
set -e
cd "$(dirname "$0")/.."
mkdir -p tune
b() { python -m paper_2005_13014_b200.build --out=tune/$1.so "${@:2}" > /dev/null; echo "$1 ${@:2}"; }
b h_2_8_3_6  -DHD_V=2 -DHD_JB=8 -DHD_S=3 -DHD_NW=6 &
b h_2_16_2_5 -DHD_V=2 -DHD_JB=16 -DHD_S=2 -DHD_NW=5 &
b h_2_8_2_8  -DHD_V=2 -DHD_JB=8 -DHD_S=2 -DHD_NW=8 &
b h_4_8_2_5  -DHD_V=4 -DHD_JB=8 -DHD_S=2 -DHD_NW=5 &
wait
b h_1_16_3_8  -DHD_V=1 -DHD_JB=16 -DHD_S=3 -DHD_NW=8 &
b h_2_12_2_6  -DHD_V=2 -DHD_JB=12 -DHD_S=2 -DHD_NW=6 &
b v_t6   -DVT_S=6 &
b v_t8   -DVT_S=8 &
wait
b v_t4   -DVT_S=4 &
b v_smem -DVA_NO_TMEM -DVA_NC=64 -DVA_LB=4 -DVA_S=3 &
wait
