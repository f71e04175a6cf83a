#!/bin/bash
# Blackwell-native instruction counts per librf_cuda kernel (UTC*MMA = tcgen05.mma,
# LDTM/STTM = tcgen05.ld/st, UTMALDG/UTMASTG = TMA tensor load/store, UBLKCP = bulk copy).
#   bash tools/sass_summary.sh > profiles/r2_sass_summary.txt
lib=${1:-paper_2603_10026_b200/librf_cuda.so}
cuobjdump -sass "$lib" | awk '
/Function :/ { if (name != "") report(); name = $3; delete c; next }
{ for (i = 1; i <= NF; ++i) { op = $i; sub(/\..*/, "", op);
    if (op ~ /^(UTCHMMA|UTCQMMA|UTCOMMA|UTCBAR|LDTM|STTM|UTMALDG|UTMASTG|UBLKCP|UTCATOMSWS|MUFU|FFMA2|FMUL2|HMMA)$/) { c[op]++; break } } }
function report() { s = ""; for (k in c) s = s " " k "=" c[k]; printf "%s:%s\n", name, s }
END { if (name != "") report() }' | sed 's/_ZN2rf[0-9A-Za-z_]*GLOBAL__N__[0-9a-f]*_[0-9]*_//' | sort
