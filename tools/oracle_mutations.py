"""Mutation check of the oracle's pins (TEST INFRASTRUCTURE).

Each mutation is a plausible mistake in oracle/gdraa_oracle.c -- a dropped term, a wrong
sign or order, a truncating cast, a reciprocal instead of a division.  The mutated source
is compiled to a temporary library (the tree is not touched), the CPU pin suite
(tests/test_oracle_pins.py) runs against it through GDRAA_ORACLE_LIB, and the mutation
must fail at least one pin.  Writes one JSON line per mutation and a summary.

    python tools/oracle_mutations.py [out.jsonl]     # default profiles/r62_oracle_mutations.jsonl
"""
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "gdraa_oracle.c")
sys.path.insert(0, ROOT)
from oracle.build import CFLAGS  # noqa: E402

# (name, exact text in gdraa_oracle.c, replacement, how many occurrences to replace)
MUTATIONS = [
    ("mean bf16 output truncates instead of RNE (P:169, AMB-13)",
     "((uint16_t *)out)[i] = oracle_f32_to_bf16_rne(m);",
     "{ uint32_t u_; memcpy(&u_, &m, 4); ((uint16_t *)out)[i] = (uint16_t)(u_ >> 16); }", 1),
    ("bf16 helper truncates (AMB-13)",
     "u += 0x7FFFu + ((u >> 16) & 1u);", "", 1),
    ("bf16 helper rounds ties away from zero",
     "u += 0x7FFFu + ((u >> 16) & 1u);", "u += 0x8000u;", 1),
    ("bf16 widening shifts by 15",
     "uint32_t u = (uint32_t)b << 16;", "uint32_t u = (uint32_t)b << 15;", 1),
    ("fold in descending rank (AMB-2)",
     """    float s = load_elem(dtype, in[0], i);
    for (int p = 1; p < N; p++) {
        float x = load_elem(dtype, in[p], i);""",
     """    float s = load_elem(dtype, in[N - 1], i);
    for (int p = N - 2; p >= 0; p--) {
        float x = load_elem(dtype, in[p], i);""", 1),
    ("fold starts from +0.0 (AMB-3)",
     "    float s = load_elem(dtype, in[0], i);\n    for (int p = 1; p < N; p++) {",
     "    float s = 0.0f;\n    for (int p = 0; p < N; p++) {", 1),
    ("reciprocal multiply instead of division (AMB-2)",
     "float m = s / (float)N;", "float m = s * (1.0f / (float)N);", 1),
    ("sum, not mean (dropped 1/N)",
     "float m = s / (float)N;", "float m = s;", 1),
    ("dropped last rank from the fold",
     "for (int p = 1; p < N; p++) {", "for (int p = 1; p < N - 1; p++) {", 1),
    ("fused multiply-add in the momentum update (AMB-4)",
     "        float t = mom * v[i];\n        float vn = t + m;",
     "        float vn = fmaf(mom, v[i], m);", 1),
    ("update adds instead of subtracts (P:157)",
     "        float wn = w[i] - u;\n        v[i] = vn;\n        w[i] = wn;\n    }\n    return 0;",
     "        float wn = w[i] + u;\n        v[i] = vn;\n        w[i] = wn;\n    }\n    return 0;", 1),
    ("update uses the old momentum",
     "        float u = lr * vn;\n        float wn = w[i] - u;\n        v[i] = vn;\n        w[i] = wn;\n    }\n    return 0;",
     "        float u = lr * v[i];\n        float wn = w[i] - u;\n        v[i] = vn;\n        w[i] = wn;\n    }\n    return 0;", 1),
    ("momentum not applied (mom ignored)",
     "        float t = mom * v[i];\n        float vn = t + m;\n        float u = lr * vn;\n        float wn = w[i] - u;\n        v[i] = vn;\n        w[i] = wn;\n    }\n    return 0;",
     "        float t = v[i];\n        float vn = t + m;\n        float u = lr * vn;\n        float wn = w[i] - u;\n        v[i] = vn;\n        w[i] = wn;\n    }\n    return 0;", 1),
    ("weight decay sign flipped (S:412)",
     "            ge = m + d;", "            ge = m - d;", 1),
    ("weight decay dropped", "            ge = m + d;", "            ge = m;", 1),
    ("weight decay on the updated weight",
     "            float d = wd * w[i];", "            float d = wd * (w[i] - lr * m);", 1),
    ("model copy truncated to bf16",
     "((uint16_t *)model)[i] = oracle_f32_to_bf16_rne(wn);",
     "{ uint32_t u_; memcpy(&u_, &wn, 4); ((uint16_t *)model)[i] = (uint16_t)(u_ >> 16); }", 1),
    ("partition without Q rounding (AMB-8)",
     "uint64_t blk = ((c + Q - 1) / Q) * Q;", "uint64_t blk = c;", 1),
    ("partition floor instead of ceil (P:162)",
     "uint64_t c = (L + (uint64_t)N - 1) / (uint64_t)N;", "uint64_t c = L / (uint64_t)N;", 1),
    ("partition offset not clamped to L",
     "    if (o > L) o = L;\n    uint64_t l = blk;", "    uint64_t l = blk;", 1),
    ("Lemma 1 bytes count the own block too (Eq. 1)",
     "out->rs_sent = (uint64_t)s_g * (L - len);", "out->rs_sent = (uint64_t)s_g * L;", 1),
    ("Lemma 2 adds per element N instead of N-1 (Eq. 3)",
     "out->adds = n1 * len;", "out->adds = (uint64_t)N * len;", 1),
    ("poly lr ignores the power (P:246)",
     "return (float)((double)lr0 * pow(frac, (double)power));",
     "return (float)((double)lr0 * frac);", 1),
    ("poly lr off by one iteration",
     "double frac = 1.0 - (double)iter / (double)max_iter;",
     "double frac = 1.0 - (double)(iter + 1) / (double)max_iter;", 1),
]


def build(src_text, out):
    with tempfile.NamedTemporaryFile("w", suffix=".c", dir=os.path.dirname(SRC),
                                     delete=False) as f:
        f.write(src_text)
        path = f.name
    try:
        subprocess.run(["gcc", *[c for c in CFLAGS if c != "-Werror"], path, "-o", out, "-lm"],
                       check=True, capture_output=True, text=True)
    finally:
        os.unlink(path)


def run_pins(lib):
    env = dict(os.environ, GDRAA_ORACLE_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q",
                        "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    failed = int(m.group(1)) if (m := re.search(r"(\d+) failed", tail)) else 0
    passed = int(m.group(1)) if (m := re.search(r"(\d+) passed", tail)) else 0
    names = sorted({l.split("::")[1].split(" ")[0].split("[")[0]
                    for l in r.stdout.splitlines() if l.startswith("FAILED")})
    return failed, passed, names, tail


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        ROOT, "profiles", "r62_oracle_mutations.jsonl")
    src = open(SRC).read()
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    lines = []
    base = os.path.join(tmp, "base.so")
    build(src, base)
    f0, p0, _, tail0 = run_pins(base)
    lines.append({"mutation": None, "failed": f0, "passed": p0, "note": "unmutated oracle"})
    caught = 0
    for name, old, new, count in MUTATIONS:
        n = src.count(old)
        if n < count:
            lines.append({"mutation": name, "error": f"pattern found {n} times"})
            continue
        lib = os.path.join(tmp, "mut.so")
        build(src.replace(old, new, count), lib)
        failed, passed, names, tail = run_pins(lib)
        caught += failed > 0
        lines.append({"mutation": name, "failed": failed, "passed": passed,
                      "failing_pins": names})
        print(f"{'CAUGHT' if failed else 'MISSED'} {failed:3d}  {name}", flush=True)
    summary = {"summary": True, "mutations": len(MUTATIONS), "caught": caught,
               "unmutated_failures": f0}
    with open(out_path, "w") as f:
        for l in lines + [summary]:
            f.write(json.dumps(l) + "\n")
    print(json.dumps(summary))
    return 0 if caught == len(MUTATIONS) and f0 == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
