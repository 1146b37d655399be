"""Per-kernel SASS instruction-class summary of libhdpstereo.so (cuobjdump):
instruction count by class, and the sm_100a features present (bulk copies /
TMA: UBLKCP / UTMALDG; mbarrier: SYNCS; tensor cores: UTC*MMA -- none expected,
nothing here is a contraction).
usage: python tools/sass_summary.py [LIB]"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1509_08197_b200/libhdpstereo.so"
want = ["k_up_chunk", "k_down_chunk", "k_seg_up", "k_seg_down", "k_ecost_range_u", "k_grp", "k_prior",
        "k_mst_coop", "k_rank_jump_async", "k_keys_finish"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
classes = {"FP32": r"^(FADD|FMUL|FFMA|FMNMX|FSEL|FSETP|FCHK|MUFU|FADD2|FFMA2|FMUL2)",
           "FP64": r"^(DADD|DMUL|DFMA|DSETP|DMNMX)", "INT": r"^(IMAD|IADD|IADD3|LEA|ISETP|LOP3|SHF|SEL|VIADD|VIMNMX|IMNMX|POPC|FLO|PRMT)",
           "LD/ST global": r"^(LDG|STG|RED|ATOM)", "shared": r"^(LDS|STS|ATOMS|LDSM)",
           "bulk/TMA": r"^(UBLKCP|UTMALDG|UTMASTG|UBLKRED)", "mbarrier": r"^SYNCS",
           "tensor": r"^(UTC|HMMA|IMMA)", "control": r"^(BRA|BSSY|BSYNC|EXIT|RET|CALL|BAR|WARPSYNC|ISBERRIES|YIELD)",
           "shuffle/vote": r"^(SHFL|VOTE|MATCH|REDUX)"}
blocks = re.split(r"\n\s*Function : ", sass)
print(f"{'kernel':<46}" + "".join(f"{c:>13}" for c in classes) + f"{'total':>8}")
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    short = re.sub(r"^_ZN3hdp", "", name)
    if not any(w in name for w in want):
        continue
    cnt = collections.Counter()
    total = 0
    for ln in b.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
        if not m:
            continue
        op = m.group(2).split(".")[0]
        total += 1
        for c, pat in classes.items():
            if re.match(pat, op):
                cnt[c] += 1
                break
    print(f"{short[:46]:<46}" + "".join(f"{cnt[c]:>13}" for c in classes) + f"{total:>8}")
