#!/bin/bash
cd "$(dirname "$0")/.."
AB_WL=cfg4_k64_f64 AB_B=64 bash scripts/gpu_ab.sh build_var/libpf16.so build_var/libpf32.so build_var/libpf48.so
AB_WL=cfg4_k128_f64 AB_B=64 bash scripts/gpu_ab.sh build_var/libpf16.so build_var/libpf32.so build_var/libpf48.so
