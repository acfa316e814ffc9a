#!/bin/bash
# SASS mnemonic evidence for the sm_100a kernels of libconvq.so (B200_PROFILING.md
# "What proves a Blackwell-native kernel"): tcgen05.mma -> UTCIMMA (2CTA = cta_group::2),
# TMA -> UTMALDG / UTMASTG / UBLKCP, tcgen05.ld -> LDTM, commit -> UTCBAR; the
# epilogue's packed conversions F2IP.S8 / I2IP.S4 and FFMA2; no legacy HMMA.
# Usage: scripts/sass_summary.sh [lib] > profiles/r02_sass_summary.txt
LIB=${1:-paper_2202_06819_b200/libconvq.so}
T=$(mktemp)
cuobjdump -sass "$LIB" > "$T"
echo "# cuobjdump -sass $LIB ($(grep -c 'Function :' "$T") kernels, arch $(grep -m1 -o 'arch = sm_[0-9a-z]*' "$T"))"
for m in "UTCIMMA" "UTCIMMA.2CTA" "UTMALDG.4D.IM2COL" "UTMALDG.4D" "UTMALDG.2D" "UTMASTG.2D" "UBLKCP" "LDTM" \
         "UTCBAR" "UTCBAR.2CTA.MULTICAST" "F2IP.S8" "I2IP.S4" "FFMA2" "VIMNMX" "HMMA" "IMMA.16" "HGMMA"; do
  printf "%-24s %8d lines\n" "$m" "$(grep -c "$m" "$T")"
done
echo "# kernels containing UTCIMMA:"
awk '/Function :/{f=$3} /UTCIMMA/{if(!(f in s)){s[f]=1; n++}} END{print n}' "$T"
rm -f "$T"
