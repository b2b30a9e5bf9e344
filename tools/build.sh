#!/bin/bash
# rebuild libipdg.so and show register / spill summary for k_sipdg<N>
cd /root/repo && python -c "
import sys; sys.path.insert(0,'.')
import __graft_entry__ as g; g.build()" 2>&1 | tail -2
grep -B1 -A2 "Compiling entry.*k_sipdgILi${1:-4}" paper_1801_00246_b200/csrc/ptxas_info.txt | grep -E "Used|spill" | sed 's/ptxas info    : //' | cut -c1-100
