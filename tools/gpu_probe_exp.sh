for e in 0 1 2 3; do TQ_JIT_DEFS=TQ_EXP=$e python tools/probe_exp.py --sf 10 2>&1 | tail -1; done
