"""One-off source transform used once to move decode-path kernels onto
programmatic dependent launch: insert pdl_enter() at the top of the named
__global__ kernels and turn their `k<<<g, b, s, st>>>(args);` launches into
launch_pdl(k, dim3(g), dim3(b), s, st, args). python tools/dev/pdl_convert.py file.cu name..."""
import re
import sys


def balanced(s, i, open_c="(", close_c=")"):
    depth = 0
    for j in range(i, len(s)):
        if s[j] == open_c:
            depth += 1
        elif s[j] == close_c:
            depth -= 1
            if depth == 0:
                return j
    raise ValueError("unbalanced")


def split_top(s):
    out, depth, cur = [], 0, ""
    for ch in s:
        if ch in "([{":
            depth += 1
        elif ch in ")]}":
            depth -= 1
        if ch == "," and depth == 0:
            out.append(cur.strip())
            cur = ""
        else:
            cur += ch
    out.append(cur.strip())
    return out


def main(path, names):
    s = open(path).read()
    for name in names:
        # kernel definitions
        for m in list(re.finditer(r"__global__[^;{]*?\b" + re.escape(name) + r"\s*\(", s)):
            pass
        pos = 0
        while True:
            m = re.search(r"__global__[^;{]*?\b" + re.escape(name) + r"\s*\(", s[pos:])
            if not m:
                break
            a = pos + m.end() - 1
            b = balanced(s, a)
            brace = s.index("{", b)
            if "pdl_enter();" not in s[brace:brace + 40]:
                s = s[:brace + 1] + "\n    pdl_enter();" + s[brace + 1:]
            pos = brace + 1
        # launches
        pos = 0
        while True:
            m = re.search(r"\b" + re.escape(name) + r"(<[^<>]*>)?\s*<<<", s[pos:])
            if not m:
                break
            st = pos + m.start()
            lt = pos + m.end()
            gt = s.index(">>>", lt)
            cfg = split_top(s[lt:gt])
            if len(cfg) == 3:
                cfg.append("0")
            g, bl, sm, stream = cfg
            ap = s.index("(", gt + 3)
            ae = balanced(s, ap)
            args = s[ap + 1:ae]
            semi = s.index(";", ae)
            kname = name + (m.group(1) or "")
            new = (f"if (int rc_ = launch_pdl({kname}, dim3({g}), dim3({bl}), {sm}, {stream}, {args.strip()})) "
                   f"return rc_;")
            s = s[:st] + new + s[semi + 1:]
            pos = st + len(new)
    open(path, "w").write(s)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
