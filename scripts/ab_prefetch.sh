set -e
./scripts/mb_tma.bin
for v in pf0 pf2 pf6; do echo "== $v"; DECATTN_LIB=paper_2604_00028_b200/lib/variants/libdecattn_$v.so python scripts/probe_timing.py 2>&1 | grep -E "L=    (64|192|512) .*(guarded|seq_aware|fixed     s=  1 )" | head -12; done
echo "== pf1 (default)"; python scripts/probe_timing.py 2>&1 | grep -E "L=    (64|192|512) .*(guarded|seq_aware|fixed     s=  1 )" | head -12
