#!/bin/bash
S="4:0:512 4:512:512 2:1024:512 1:1500:512"
for t in 0 1; do echo "== TC $t"; TLT_ATTN_TC=$t timeout 200 python tools/probe_attn.py $S; done
