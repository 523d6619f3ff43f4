"""Measurement / policy harness around the C ABI (rec_serve): SLA-bounded QPS search and
Hercules' Algorithm 1 over the serving policy.  Not a step of the hot path; never imports
the oracle."""
