#!/bin/bash
# tuning builds of liboec for the f32 vadv solver tiles (VF_NC, VF_LB, VF_S) into tune/
set -e
cd "$(dirname "$0")/.."
mkdir -p tune
b() { python -m paper_2005_13014_b200.build --out=tune/$1.so "${@:2}" > /dev/null; echo "$1 ${@:2}"; }
b f_32_4_4 -DVF_NC=32 -DVF_LB=4 -DVF_S=4 &
b f_32_8_4 -DVF_NC=32 -DVF_LB=8 -DVF_S=4 &
b f_64_4_6 -DVF_NC=64 -DVF_LB=4 -DVF_S=6 &
b f_64_8_4 -DVF_NC=64 -DVF_LB=8 -DVF_S=4 &
wait
b f_64_8_3 -DVF_NC=64 -DVF_LB=8 -DVF_S=3 &
b f_128_4_4 -DVF_NC=128 -DVF_LB=4 -DVF_S=4 &
b f_32_4_8 -DVF_NC=32 -DVF_LB=4 -DVF_S=8 &
b f_32_8_6 -DVF_NC=32 -DVF_LB=8 -DVF_S=6 &
wait
