#!/bin/bash
# spill_map.sh <object> <kernel-substring>: SASS line numbers of local-memory traffic, barriers,
# REDUX and back-edges of one kernel (to see whether spills sit inside the per-column loop)
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{f=($0 ~ pat)} f' | grep -E "^\s+/\*[0-9a-f]+\*/" > /tmp/_k.sass
echo "instructions: $(wc -l < /tmp/_k.sass)"
grep -n "STL\|LDL\|BAR.SYNC\|REDUX\|MUFU.RCP64H\|EXIT" /tmp/_k.sass | awk '{$NF=""; print}' | cut -c1-70
grep -n "BRA" /tmp/_k.sass | awk '{ if ($0 ~ /0xffff/) print "backedge " $0 }' | cut -c1-80
