"""Device time per kernel name from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections, csv, sys


def main(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    t, n = collections.Counter(), collections.Counter()
    for r in rows:
        name = r[4].split("(")[0]
        t[name] += float(r[14].replace(",", "")) / 1e6
        n[name] += 1
    tot = sum(t.values())
    print(f"# device time per kernel from {title} (ncu launch list, serialised, cold-cache)")
    for k, v in t.most_common():
        print(f"{k:44s} {v:9.3f} ms  {100 * v / tot:5.1f}%  launches {n[k]}")
    print(f"{'total':44s} {tot:9.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
