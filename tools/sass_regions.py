"""Static SASS size per source region of one kernel (nvdisasm -g output)."""
import re
import sys


def sizes(sass_path, func_substr, src_name):
    lines = open(sass_path).read().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and func_substr in l)
    cur_file, cur_line = "", 0
    per_line = {}
    for l in lines[start + 1:]:
        if l.startswith("//---------------------") and ".text." in l:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur_file, cur_line = m.group(1), int(m.group(2))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
            key = cur_line if cur_file.endswith(src_name) else "other:" + cur_file.split("/")[-1]
            per_line[key] = per_line.get(key, 0) + 1
    return per_line


if __name__ == "__main__":
    pl = sizes(sys.argv[1], sys.argv[2], "decode.cu")
    src = open("paper_1809_03606_b200/csrc/decode.cu").read().split("\n")
    tot = sum(pl.values())
    print("total SASS instructions", tot, "=", tot * 16 // 1024, "KB")
    for k, v in sorted(pl.items(), key=lambda x: -x[1])[:40]:
        txt = src[k - 1].strip()[:90] if isinstance(k, int) else ""
        print(f"{v:5d} {k!s:>24} | {txt}")
