for pb in 1 2; do for bl in 1 0; do
TQ_BLOOM=$bl TQ_JIT_DEFS=TQ_PB=$pb python tools/probe_exp.py --sf 10 2>&1 | tail -1
done; done
