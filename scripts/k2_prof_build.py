"""Build variants/prof.so: K2 with clock64 phase stamps (admission, live prefix,
candidate parameters, decide, commit) printed for block 0 / segment 0.
The source tree is restored afterwards."""
import os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
p = os.path.join(ROOT, "paper_2605_05527_b200", "csrc", "k2_replay.cu")
orig = open(p).read()
s = orig
def ins(before, text):
    global s
    assert before in s, before
    s = s.replace(before, text + before, 1)
ins('      if (active && status == ES_OK && ++iters > 2u * total + 4u) status = ES_ERR_INTERNAL;', '      long long T0 = clock64();\n')
ins('      const bool go = run && status == ES_OK;', '      long long T1 = clock64();\n')
ins('      const Cand cand = cand_params<LPS, MM>(sg, P, C, len, wmax);', '      long long T2 = clock64();\n')
ins('      const uint32_t tt = t;\n', '      long long T3 = clock64();\n')
ins('      // a8: commit', '      long long T4 = clock64();\n')
ins('      if (__any_sync(FULL, active && (served >= total || status != ES_OK))) break;',
    '      long long T5 = clock64();\n      if (dec) { pf[0] += T1 - T0; pf[1] += T2 - T1; pf[2] += T3 - T2; pf[3] += T4 - T3; pf[4] += T5 - T4; pf[5]++; }\n')
ins('  for (;;) {\n    // ---- refill', '  long long pf[6] = {0, 0, 0, 0, 0, 0};\n')
old = '''      active = false;
    }
  }
}'''
assert old in s
s = s.replace(old, '''      active = false;
    }
  }
  if (pf[5] > 0 && sg.sl == 0 && blockIdx.x == 0)
    printf("K2PROF decisions %lld cycles/decision: admission %lld, prefix %lld, cand %lld, decide %lld, commit %lld\\n",
           pf[5], pf[0] / max(pf[5], 1ll), pf[1] / max(pf[5], 1ll), pf[2] / max(pf[5], 1ll),
           pf[3] / max(pf[5], 1ll), pf[4] / max(pf[5], 1ll));
}''')
s = s.replace('#include <cstdlib>', '#include <cstdio>\n#include <cstdlib>')
try:
    open(p, "w").write(s)
    sys.path.insert(0, os.path.join(ROOT, "paper_2605_05527_b200"))
    import build
    os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
    build.build(force=True, lib=os.path.join(ROOT, "variants", "prof.so"))
finally:
    open(p, "w").write(orig)
