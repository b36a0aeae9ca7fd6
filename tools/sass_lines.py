"""Static SASS instruction count per source line for one kernel (needs
-lineinfo): python tools/sass_lines.py <nvdisasm -g -c output> <mangled-name-substring> [top]"""
import collections
import re
import sys

txt = open(sys.argv[1]).read()
start = txt.find(".text." + sys.argv[2]) if not sys.argv[2].startswith(".text.") else txt.find(sys.argv[2])
start = txt.find("\n", start)
end = txt.find("//---------------------", start + 10)
body = txt[start:end]
cur, cnt, ops = None, collections.Counter(), collections.defaultdict(collections.Counter)
for line in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        cnt[cur] += 1
        ops[cur][m.group(2)] += 1
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:top]:
    print(v, k, dict(ops[k].most_common(4)))
print("total", sum(cnt.values()))
