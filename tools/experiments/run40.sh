for t in 8x8 8x4 4x8 6x8; do for P in 1 2 3; do for o in 0 5; do
K="IAAT_FORCE_FAMILY=5 IAAT_FORCE_TILE=$t IAAT_FORCE_ORDER=$o IAAT_FORCE_P=$P IAAT_FORCE_CTAS=1"
echo "ksw $t P$P o$o: $(env $K python tools/run_case.py f32 NN 64 64 64 --reps 8 --plan 2>&1 | python3 -c 'import sys; L=sys.stdin.read().splitlines(); import json; p=json.loads(L[0].replace("\x27","\"").replace("True","true").replace("False","false")) if L[0].startswith("{") else {}; print(p.get("family"), p.get("compute_warps"), L[-1])')"
done; done; done
