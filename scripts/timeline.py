"""Per-layer critical-chain breakdown from a MOEPIC_TIMELINE dump (tools only).

    MOEPIC_TIMELINE=/tmp/tl.jsonl python bench.py --config qwen3 --prefetch-window-us 0 ...
    python scripts/timeline.py /tmp/tl.jsonl [--skip 200] [--link-gbs 55.6]

For consecutive decode layer steps i -> i+1 (times in microseconds, medians over the steps):
  copy_done(i) -> K2 final start      the final K2 waits for the last on-demand copy
  K2 final                            in-kernel span (first CTA start .. last CTA end)
  K2 final end -> router(i+1) start   launch gap (PDL or plain)
  router(i+1)                         in-kernel span
  router start -> host sees routing   (router up to the routing words + mailbox poll)
  routing seen -> first copy issued   host classification / plan bookkeeping
  first copy issued -> copy stream    a one-thread stamp kernel on the copy stream right before the
                                      first on-demand copy: when the stream gets to the copies
  first copy issued -> first byte     estimated: copy_done(i+1) - od_bytes(i+1) / link rate
  link idle                           first byte(i+1) - copy_done(i)
"""
import argparse
import json
import statistics


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--skip", type=int, default=0, help="ignore the first records (adaptation / warm-up)")
    ap.add_argument("--link-gbs", type=float, default=55.6)
    a = ap.parse_args()
    recs = [json.loads(x) for x in open(a.path) if x.strip()][a.skip:]
    rows = {k: [] for k in ("wait_k2", "k2_final", "k2_to_router", "router", "router_to_seen", "seen_to_issue",
                            "issue_to_copy_stream", "copy_stream_to_byte", "issue_to_byte", "link_idle", "od_us")}
    for r, n in zip(recs, recs[1:]):
        cd, fs, fe = r["copy_done"], r["k2_final"][0], r["k2_final"][1]
        rs, re_ = n["router"]
        seen, first_issue = n["host"][1], n["host"][2]
        ncd = n["copy_done"]
        if min(cd, fs, fe, rs, re_, ncd) < 0 or first_issue <= 0 or n["od_bytes"] == 0:
            continue
        od_us = n["od_bytes"] / (a.link_gbs * 1e3)
        first_byte = ncd - od_us * 1e3
        rows["wait_k2"].append((fs - cd) / 1e3)
        rows["k2_final"].append((fe - fs) / 1e3)
        rows["k2_to_router"].append((rs - fe) / 1e3)
        rows["router"].append((re_ - rs) / 1e3)
        rows["router_to_seen"].append((seen - rs) / 1e3)
        rows["seen_to_issue"].append((first_issue - seen) / 1e3)
        rows["issue_to_byte"].append((first_byte - first_issue) / 1e3)
        if n.get("copy_start", -1) > 0:
            rows["issue_to_copy_stream"].append((n["copy_start"] - first_issue) / 1e3)
            rows["copy_stream_to_byte"].append((first_byte - n["copy_start"]) / 1e3)
        rows["link_idle"].append((first_byte - cd) / 1e3)
        rows["od_us"].append(od_us)
    print(f"{len(rows['link_idle'])} layer transitions")
    for k, v in rows.items():
        if v:
            print(f"  {k:16s} median {statistics.median(v):8.1f} us   mean {statistics.mean(v):8.1f}")


if __name__ == "__main__":
    main()
