"""Reference-side integration: the binding a tnkit maintainer would add (tnkit_b200) and
the harness that runs tnkit's own test suite with that binding installed."""
